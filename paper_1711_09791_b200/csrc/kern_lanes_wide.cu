// Instantiates the widths 11..21 (r = 5..10) kernels of the two-pass modes (r = 11..15:
// kern_lanes_wide2.cu): the
// generic TMA producer + the lane-strided consumer (kernels.cuh,
// consume_item_lanes), any row alignment. The single pass is in
// kern_lanes_wide_single.cu (one TU per family keeps nvcc builds parallel).
#include "kernels.cuh"
#include "launch.h"

namespace sc {

// symw: mirror-symmetric taps (w[j] == w[2r-j] bitwise): products shared by value;
// aligned: 16-B aligned rows -> the adjacent-column consumer (consume_item_adj)
const void* kernel_lanes_wide(int mode, int rad, bool symw, bool aligned) {
#define SC_KA(R, A)                                                                                   \
    switch (mode) {                                                                                   \
        case MODE_FUSED:                                                                              \
            return symw ? (const void*)sepconv_lanes_wide_kernel<MODE_FUSED, R, 1, A>                 \
                        : (const void*)sepconv_lanes_wide_kernel<MODE_FUSED, R, 0, A>;                \
        case MODE_HPASS: return (const void*)sepconv_lanes_wide_kernel<MODE_HPASS, R, 0, A>;          \
        case MODE_VPASS: return (const void*)sepconv_lanes_wide_kernel<MODE_VPASS, R, 0, A>;          \
        default: return nullptr;                                                                      \
    }
#define SC_K(R)            \
    case R:                \
        if (aligned) {     \
            SC_KA(R, true) \
        }                  \
        SC_KA(R, false)
    switch (rad) {
        SC_K(5)
        SC_K(6)
        SC_K(7)
        SC_K(8)
        SC_K(9)
        SC_K(10)
        default:
            return nullptr;
    }
#undef SC_K
#undef SC_KA
}

}  // namespace sc
