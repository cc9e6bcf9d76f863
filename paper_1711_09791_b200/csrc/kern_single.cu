// Instantiates the row-streaming kernel for MODE_SINGLE (one TU per mode keeps
// nvcc builds parallel). See kernels.cuh.
#include "kernels.cuh"
#include "direct.cuh"
#include "launch.h"

namespace sc {

// sym: 0 none, 1 mirror-symmetric rows (K[i][j] == K[2r-i][j]), 2 rows and columns
const void* kernel_single(int rad, bool aligned, int sym) {
    // symmetric-tap variants exist for r >= 1 (r = 0 has a single tap)
    if (rad < 1) sym = 0;
#define SC_KA(R, S)                                                                       \
    return aligned ? (const void*)sepconv_rows_kernel<MODE_SINGLE, R, true, (R >= 1 ? S : 0)> \
                   : (const void*)sepconv_rows_kernel<MODE_SINGLE, R, false, (R >= 1 ? S : 0)>;
#define SC_K(R)                       \
    case R:                           \
        if (sym == 2) SC_KA(R, 2)     \
        if (sym == 1) SC_KA(R, 1)     \
        SC_KA(R, 0)
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
#undef SC_KA
}

// Single pass + in-place copy-back in one pass (aligned rows only).
const void* kernel_single_cb(int rad, int sym) {
    if (rad < 1) sym = 0;
#define SC_KS(R, S) return (const void*)sepconv_rows_kernel<MODE_SINGLECB, R, true, (R >= 1 ? S : 0)>;
#define SC_K(R)                   \
    case R:                       \
        if (sym == 2) SC_KS(R, 2) \
        if (sym == 1) SC_KS(R, 1) \
        SC_KS(R, 0)
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
#undef SC_KS
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
