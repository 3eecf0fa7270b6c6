// ts_cstream_w16.cu -- instantiations of k_cstream with 16 walker warps.
#include "ts_cstream_kernel.cuh"

namespace ts {
namespace cstream_detail {

cudaError_t launch_w16(const CStreamArgs &a, int device, cudaStream_t stream) {
    if (a.B == 128 && a.k == 8) return launch_kgw<8, 4, 16>(a, device, stream);
    if (a.B == 128 && a.k == 4) return launch_kgw<4, 4, 16>(a, device, stream);
    if (a.B == 64 && a.k == 8) return launch_kgw<8, 2, 16>(a, device, stream);
    if (a.B == 32 && a.k == 8) return launch_kgw<8, 1, 16>(a, device, stream);
    if (a.B == 64 && a.k == 4) return launch_kgw<4, 2, 16>(a, device, stream);
    if (a.B == 64 && a.k == 3) return launch_kgw<3, 2, 16>(a, device, stream);
    if (a.B == 32 && a.k == 4) return launch_kgw<4, 1, 16>(a, device, stream);
    if (a.B == 32 && a.k == 3) return launch_kgw<3, 1, 16>(a, device, stream);
    if (a.B == 32 && a.k == 2) return launch_kgw<2, 1, 16>(a, device, stream);
    return cudaErrorInvalidConfiguration;
}

}  // namespace cstream_detail
}  // namespace ts
