// fc2_inst_b5.cu -- fast-path kernel instantiations for 5-bit codes.
#include "fc2_kernels.cuh"

namespace fc2 {
FC2_INSTANTIATE_B(5)
}  // namespace fc2
