// Width instantiations of the K1/K2 tile kernel (split for parallel compilation).
#include "knn_tile.cuh"

namespace cmb {
namespace knn_detail {
template cudaError_t launch_tile_w<1>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<2>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<3>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<4>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<5>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<6>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<7>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<8>(const KnnArgs&, int, cudaStream_t);
}  // namespace knn_detail
}  // namespace cmb
