// ts_rank_i1.cu -- explicit instantiations of the rank walk launchers.
#include "ts_rank_kernel.cuh"

namespace ts {
namespace rank_detail {
template cudaError_t launch_rank_d<8>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<9>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<10>(const RankArgs &, int, int, cudaStream_t);
}  // namespace rank_detail
}  // namespace ts
