// tc_prefill.cuh — placeholder until the tcgen05 prefill kernel lands.
#pragma once
#include "tc_kernels.hpp"

namespace bsra {
inline int tc_prefill_launch(const AttnParams&, const TcLaunch&, cudaStream_t, const char**, const char** why, int) {
  *why = "tcgen05 prefill kernel not built yet";
  return 0;
}
}  // namespace bsra
