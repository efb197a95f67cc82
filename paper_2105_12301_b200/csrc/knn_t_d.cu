// Width instantiations of the K1/K2 tile kernel (split for parallel compilation).
#include "knn_tile.cuh"

namespace cmb {
namespace knn_detail {
template cudaError_t launch_tile_w<18>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<19>(const KnnArgs&, int, cudaStream_t);
template cudaError_t launch_tile_w<20>(const KnnArgs&, int, cudaStream_t);
}  // namespace knn_detail
}  // namespace cmb
