// fc2_inst_b3.cu -- fast-path kernel instantiations for 3-bit codes.
#include "fc2_kernels.cuh"

namespace fc2 {
FC2_INSTANTIATE_B(3)
}  // namespace fc2
