// tc_kernels.hpp — launch entry for the tcgen05 (5th-gen tensor core) attention kernels.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace bsra {

struct TcLaunch {
  bool f16 = false;        // fp16 inputs (else bf16)
  int T_q = 0;             // plan tile
  int grid = 0;            // persistent grid (= plan num_ctas)
  int64_t total_qo = 0;    // rows of the q tensor map (the plan's sum of l_qo; max_total_qo_rows under capture)
  int align = 0;           // chunk alignment in tokens
  int page_size = 0;
  int kc = 16;             // decode: live fused columns (4 / 8 / 16), from the plan or max_qo_len
  int mask = 0;
  bool pdl = false;        // programmatic dependent launch (BSRA_FLAG_PDL)
  bool ragged = false;     // contiguous KV [N, H_kv, D] (p.kv_ragged)
  int64_t total_kv = 0;    // ragged: the token extent of the k / v maps
  bool f8kv = false;       // K/V pools in E4M3 (fp8 KV cache, R28)
  bool rope = false;       // fused RoPE (R31): decode tiles only
  bool force_cp = false;   // decode: row gather even where TMA boxes apply (BSRA_FLAG_CP_GATHER)
  bool force_cp_async = false;  // row gather by cp.async even where TMA gather4 applies (tests, A/B)
};

// Launches the tcgen05 kernel for this plan if one applies (bf16/f16, D = 128, supported page
// size / group size). Returns 1 if launched, 0 if no tcgen05 kernel handles this configuration
// (*why says which condition failed), -1 on a CUDA error.
int tc_launch(const AttnParams& p, const TcLaunch& L, cudaStream_t st, const char** name, const char** why);

}  // namespace bsra
