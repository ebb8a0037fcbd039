// fc2_inst_b4.cu -- fast-path kernel instantiations for 4-bit codes.
#include "fc2_kernels.cuh"

namespace fc2 {
FC2_INSTANTIATE_B(4)
}  // namespace fc2
