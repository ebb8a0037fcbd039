// fc2_inst_b8.cu -- fast-path kernel instantiations for 8-bit codes.
#include "fc2_kernels.cuh"

namespace fc2 {
FC2_INSTANTIATE_B(8)
}  // namespace fc2
