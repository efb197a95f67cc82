// Width instantiations of the K1/K2 kernel (split for parallel compilation).
#include "knn_sweep.cuh"

namespace cmb {
namespace knn_detail {
template cudaError_t launch_w<15>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<16>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<17>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<18>(const KnnArgs&, int, cudaStream_t);
}  // namespace knn_detail
}  // namespace cmb
