// Instantiates the row-streaming kernel for MODE_VPASS (one TU per mode keeps
// nvcc builds parallel). See kernels.cuh.
#include "kernels.cuh"
#include "direct.cuh"
#include "launch.h"

namespace sc {

const void* kernel_vpass(int rad, bool aligned) {
#define SC_K(R)                                                                                   \
    case R:                                                                                       \
        return aligned ? (const void*)sepconv_rows_kernel<MODE_VPASS, R, true>                       \
                       : (const void*)sepconv_rows_kernel<MODE_VPASS, R, false>;
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

const void* kernel_vpass_direct(int rad) {
    switch (rad) {
        case 0: return (const void*)sepconv_direct_kernel<MODE_VPASS, 0>;
        case 1: return (const void*)sepconv_direct_kernel<MODE_VPASS, 1>;
        case 2: return (const void*)sepconv_direct_kernel<MODE_VPASS, 2>;
        case 3: return (const void*)sepconv_direct_kernel<MODE_VPASS, 3>;
        case 4: return (const void*)sepconv_direct_kernel<MODE_VPASS, 4>;
        default: return nullptr;
    }
}

}  // namespace sc
