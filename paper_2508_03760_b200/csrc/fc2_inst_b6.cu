// fc2_inst_b6.cu -- fast-path kernel instantiations for 6-bit codes.
#include "fc2_kernels.cuh"

namespace fc2 {
FC2_INSTANTIATE_B(6)
}  // namespace fc2
