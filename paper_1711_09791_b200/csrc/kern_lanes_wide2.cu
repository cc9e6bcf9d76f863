// Instantiates the widths 23..31 (r = 11..15) kernels of the two-pass modes (r = 5..10:
// kern_lanes_wide.cu): the
// generic TMA producer + the lane-strided consumer (kernels.cuh,
// consume_item_lanes), any row alignment. The single pass is in
// kern_lanes_wide_single.cu (one TU per family keeps nvcc builds parallel).
#include "kernels.cuh"
#include "launch.h"

namespace sc {

// symw: mirror-symmetric taps (w[j] == w[2r-j] bitwise): products shared by value
const void* kernel_lanes_wide2(int mode, int rad, bool symw) {
#define SC_K(R)                                                                                       \
    case R:                                                                                           \
        switch (mode) {                                                                               \
            case MODE_FUSED:                                                                          \
                return symw ? (const void*)sepconv_lanes_wide_kernel<MODE_FUSED, R, 1>                \
                            : (const void*)sepconv_lanes_wide_kernel<MODE_FUSED, R, 0>;               \
            case MODE_HPASS: return (const void*)sepconv_lanes_wide_kernel<MODE_HPASS, R, 0>;         \
            case MODE_VPASS: return (const void*)sepconv_lanes_wide_kernel<MODE_VPASS, R, 0>;         \
            default: return nullptr;                                                                  \
        }
    switch (rad) {
        SC_K(11)
        SC_K(12)
        SC_K(13)
        SC_K(14)
        SC_K(15)
        default:
            return nullptr;
    }
#undef SC_K
}

}  // namespace sc
