// ts_rank_i2.cu -- explicit instantiations of the rank walk launchers.
#include "ts_rank_kernel.cuh"

namespace ts {
namespace rank_detail {
template cudaError_t launch_rank_d<11>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<12>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<13>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<14>(const RankArgs &, int, int, cudaStream_t);
}  // namespace rank_detail
}  // namespace ts
