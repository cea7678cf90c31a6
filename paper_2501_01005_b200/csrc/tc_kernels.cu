#include "tc_kernels.hpp"

namespace bsra {
int tc_launch(const AttnParams&, bool, int, int, cudaStream_t, const char**) { return 0; }
}  // namespace bsra
