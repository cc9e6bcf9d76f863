// Instantiates the row-streaming kernel for MODE_FUSED (one TU per mode keeps
// nvcc builds parallel). See kernels.cuh.
#include "kernels.cuh"
#include "direct.cuh"
#include "launch.h"

namespace sc {

// symw: mirror-symmetric taps (w[j] == w[2r-j] bitwise): products shared by value;
// sig: the peer-band instantiation with the row-band readiness signalling
const void* kernel_fused(int rad, bool aligned, bool symw, bool sig) {
    if (rad < 1) symw = false;
#define SC_KF(R, S)                                                                                        \
    {                                                                                                      \
        if (sig)                                                                                           \
            return aligned ? (const void*)sepconv_rows_kernel<MODE_FUSED, R, true, (R >= 1 ? S : 0), true>  \
                           : (const void*)sepconv_rows_kernel<MODE_FUSED, R, false, (R >= 1 ? S : 0), true>; \
        return aligned ? (const void*)sepconv_rows_kernel<MODE_FUSED, R, true, (R >= 1 ? S : 0)>           \
                       : (const void*)sepconv_rows_kernel<MODE_FUSED, R, false, (R >= 1 ? S : 0)>;          \
    }
#define SC_K(R)                \
    case R:                    \
        if (symw) SC_KF(R, 1)  \
        SC_KF(R, 0)
    switch (rad) {
        SC_K(0)
        SC_K(1)
        SC_K(2)
        SC_K(3)
        SC_K(4)
        default:
            return nullptr;
    }
#undef SC_K
#undef SC_KF
}

// Split-fused (the reference's exact scratch end state in one pass; aligned rows only).
const void* kernel_splitf(int rad, bool symw) {
    switch (rad) {
        case 0: return (const void*)sepconv_rows_kernel<MODE_SPLITF, 0, true>;
        case 1: return symw ? (const void*)sepconv_rows_kernel<MODE_SPLITF, 1, true, 1>
                            : (const void*)sepconv_rows_kernel<MODE_SPLITF, 1, true>;
        case 2: return symw ? (const void*)sepconv_rows_kernel<MODE_SPLITF, 2, true, 1>
                            : (const void*)sepconv_rows_kernel<MODE_SPLITF, 2, true>;
        case 3: return symw ? (const void*)sepconv_rows_kernel<MODE_SPLITF, 3, true, 1>
                            : (const void*)sepconv_rows_kernel<MODE_SPLITF, 3, true>;
        case 4: return symw ? (const void*)sepconv_rows_kernel<MODE_SPLITF, 4, true, 1>
                            : (const void*)sepconv_rows_kernel<MODE_SPLITF, 4, true>;
        default: return nullptr;
    }
}

const void* kernel_fused_direct(int rad) {
    switch (rad) {
        case 0: return (const void*)sepconv_direct_kernel<MODE_FUSED, 0>;
        case 1: return (const void*)sepconv_direct_kernel<MODE_FUSED, 1>;
        case 2: return (const void*)sepconv_direct_kernel<MODE_FUSED, 2>;
        case 3: return (const void*)sepconv_direct_kernel<MODE_FUSED, 3>;
        case 4: return (const void*)sepconv_direct_kernel<MODE_FUSED, 4>;
        default: return nullptr;
    }
}

}  // namespace sc
