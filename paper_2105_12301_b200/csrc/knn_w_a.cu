// Width instantiations of the K1/K2 kernel (split for parallel compilation).
#include "knn_sweep.cuh"

namespace cmb {
namespace knn_detail {
template cudaError_t launch_w<1>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<2>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<3>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<4>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<5>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<6>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<7>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<8>(const KnnArgs&, int, cudaStream_t);
}  // namespace knn_detail
}  // namespace cmb
