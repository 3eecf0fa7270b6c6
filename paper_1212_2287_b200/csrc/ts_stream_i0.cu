// ts_stream_i0.cu -- explicit instantiations of the streaming kernel launchers
// (split across translation units so nvcc compiles them in parallel).
#include "ts_stream_kernel.cuh"

namespace ts {
namespace stream_detail {
template cudaError_t launch_d<0>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_ws_d<0>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_d<1>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_ws_d<1>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_d<2>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_ws_d<2>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_d<3>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_ws_d<3>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_d<4>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_ws_d<4>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_d<5>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_ws_d<5>(const StreamArgs &, int, cudaStream_t);
}  // namespace stream_detail
}  // namespace ts
