// Width instantiations of the K1/K2 kernel (split for parallel compilation).
#include "knn_sweep.cuh"

namespace cmb {
namespace knn_detail {
template cudaError_t launch_w<24>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<28>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_w<30>(const KnnArgs&, int, cudaStream_t);
}  // namespace knn_detail
}  // namespace cmb
