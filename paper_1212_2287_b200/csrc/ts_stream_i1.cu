// ts_stream_i1.cu -- explicit instantiations of the streaming kernel launchers
// (split across translation units so nvcc compiles them in parallel).
#include "ts_stream_kernel.cuh"

namespace ts {
namespace stream_detail {
template cudaError_t launch_d<6>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_ws_d<6>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_d<7>(const StreamArgs &, int, cudaStream_t);
template cudaError_t launch_ws_d<7>(const StreamArgs &, int, cudaStream_t);
}  // namespace stream_detail
}  // namespace ts
