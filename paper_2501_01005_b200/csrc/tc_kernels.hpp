// tc_kernels.hpp — launch entry for the tcgen05 (5th-gen tensor core) attention kernels.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace bsra {
// Launches the tcgen05 kernel for this tile size if one applies (bf16/f16, D = 128).
// Returns 1 if launched, 0 if no tcgen05 kernel handles this configuration, -1 on launch error.
int tc_launch(const AttnParams& p, bool bf16, int T_q, int grid, cudaStream_t st, const char** name);
}  // namespace bsra
