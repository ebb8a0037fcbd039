// fc2_inst_b7.cu -- fast-path kernel instantiations for 7-bit codes.
#include "fc2_kernels.cuh"

namespace fc2 {
FC2_INSTANTIATE_B(7)
}  // namespace fc2
