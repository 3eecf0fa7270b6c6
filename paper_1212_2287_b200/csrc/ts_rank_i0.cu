// ts_rank_i0.cu -- explicit instantiations of the rank walk launchers
// (split across translation units so nvcc compiles them in parallel).
#include "ts_rank_kernel.cuh"

namespace ts {
namespace rank_detail {
template cudaError_t launch_rank_d<1>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<2>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<3>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<4>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<5>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<6>(const RankArgs &, int, int, cudaStream_t);
template cudaError_t launch_rank_d<7>(const RankArgs &, int, int, cudaStream_t);
}  // namespace rank_detail
}  // namespace ts
