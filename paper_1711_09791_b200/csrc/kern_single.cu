// Instantiates the row-streaming kernel for MODE_SINGLE (one TU per mode keeps
// nvcc builds parallel). See kernels.cuh.
#include "kernels.cuh"
#include "direct.cuh"
#include "launch.h"

namespace sc {

const void* kernel_single(int rad, bool aligned, bool sym) {
    // symmetric-tap variants exist for r >= 1 (r = 0 has a single tap)
    sym = sym && rad >= 1;
#define SC_K(R)                                                                                   \
    case R:                                                                                       \
        if (sym)                                                                                  \
            return aligned ? (const void*)sepconv_rows_kernel<MODE_SINGLE, R, true, (R >= 1)>          \
                           : (const void*)sepconv_rows_kernel<MODE_SINGLE, R, false, (R >= 1)>;        \
        return aligned ? (const void*)sepconv_rows_kernel<MODE_SINGLE, R, true>                       \
                       : (const void*)sepconv_rows_kernel<MODE_SINGLE, R, false>;
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
}

// Single pass + in-place copy-back in one pass (aligned rows only).
const void* kernel_single_cb(int rad, bool sym) {
    sym = sym && rad >= 1;
#define SC_K(R)                                                                                          \
    case R:                                                                                              \
        return sym ? (const void*)sepconv_rows_kernel<MODE_SINGLECB, R, true, (R >= 1)>                  \
                   : (const void*)sepconv_rows_kernel<MODE_SINGLECB, R, true>;
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
}

const void* kernel_single_direct(int rad) {
    switch (rad) {
        case 0: return (const void*)sepconv_direct_kernel<MODE_SINGLE, 0>;
        case 1: return (const void*)sepconv_direct_kernel<MODE_SINGLE, 1>;
        case 2: return (const void*)sepconv_direct_kernel<MODE_SINGLE, 2>;
        case 3: return (const void*)sepconv_direct_kernel<MODE_SINGLE, 3>;
        case 4: return (const void*)sepconv_direct_kernel<MODE_SINGLE, 4>;
        default: return nullptr;
    }
}

}  // namespace sc
