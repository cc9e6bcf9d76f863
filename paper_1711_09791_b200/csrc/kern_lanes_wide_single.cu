// Instantiates the widths 11..21 (r = 5..10) single-pass kernels (wider dense folds
// spill even at 255 registers: they stay on the plain kernel of kern_wide.cu) (dense
// (2r+1)^2 fold, S/conv.py:86-114): generic TMA producer + lane-strided consumer
// (kernels.cuh, consume_item_lanes), any row alignment.
#include "kernels.cuh"
#include "launch.h"

namespace sc {

const void* kernel_lanes_wide_single(int rad) {
    switch (rad) {
        case 5: return (const void*)sepconv_lanes_wide_kernel<MODE_SINGLE, 5, 0>;
        case 6: return (const void*)sepconv_lanes_wide_kernel<MODE_SINGLE, 6, 0>;
        case 7: return (const void*)sepconv_lanes_wide_kernel<MODE_SINGLE, 7, 0>;
        case 8: return (const void*)sepconv_lanes_wide_kernel<MODE_SINGLE, 8, 0>;
        case 9: return (const void*)sepconv_lanes_wide_kernel<MODE_SINGLE, 9, 0>;
        case 10: return (const void*)sepconv_lanes_wide_kernel<MODE_SINGLE, 10, 0>;
        default: return nullptr;
    }
}

}  // namespace sc
