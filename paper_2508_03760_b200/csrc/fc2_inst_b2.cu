// fc2_inst_b2.cu -- fast-path kernel instantiations for 2-bit codes.
#include "fc2_kernels.cuh"

namespace fc2 {
FC2_INSTANTIATE_B(2)
}  // namespace fc2
