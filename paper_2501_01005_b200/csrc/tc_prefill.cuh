// tc_prefill.cuh — launch of the ragged paged prefill kernel (tc_prefill2.cuh) for tiles of
// T_q = 64 / 128 (streamed) or 256 (paired) head-fused rows: builds the TMA maps over q and the
// K/V pools and picks the instantiation (mask mode, pairing, dtype).
#pragma once
#include <cstdlib>

#include "tc_decode.cuh"
#include "tc_kernels.hpp"
#include "tc_prefill2.cuh"

namespace bsra {

bool make_q_map_ext(CUtensorMap* m, const void* q, bool f16, int H_qo, int64_t N, int hb, int tb);
bool make_kv_maps(TcParams& tp, const AttnParams& p, const TcLaunch& L, int B);

inline int tc_prefill_launch(const AttnParams& p, const TcLaunch& L, cudaStream_t st, const char** name,
                             const char** why, int B) {
  const int g = p.g;
  if (g > 128) {
    *why = "group size > 128";
    return 0;
  }
  TcParams tp;
  memset(&tp, 0, sizeof(tp));
  tp.p = p;
  tp.box_tok = B;
  tp.q_hb = g;
  tp.q_tb = 128 / g;
  tp.f16 = L.f16;
  tp.pdl = L.pdl;
#ifdef BSRA_EXPERIMENTS
  // timing experiments (scripts/trace_prefill.py); compiled out of the shipped library
  static const int dbg = getenv("BSRA_DEBUG_PREFILL") ? atoi(getenv("BSRA_DEBUG_PREFILL")) : 0;
  tp.dbg = dbg;
#endif
  if (!make_q_map_ext(&tp.tq, p.q, L.f16, p.H_qo, L.total_qo, tp.q_hb, tp.q_tb) || !make_kv_maps(tp, p, L, B)) {
    *why = "cuTensorMapEncodeTiled failed";
    return -1;
  }
  cudaError_t e;
  if (L.T_q == 256) {  // paired: both softmax WGs on one item, every K/V tile feeds 256 rows
    switch (L.mask) {
      case 0: e = launch_prefill2_t<0, true>(tp, L.grid, st); break;
      case 1: e = launch_prefill2_t<1, true>(tp, L.grid, st); break;
      default: e = launch_prefill2_t<2, true>(tp, L.grid, st); break;
    }
  } else {
    switch (L.mask) {
      case 0: e = launch_prefill2_t<0, false>(tp, L.grid, st); break;
      case 1: e = launch_prefill2_t<1, false>(tp, L.grid, st); break;
      default: e = launch_prefill2_t<2, false>(tp, L.grid, st); break;
    }
  }
  if (e != cudaSuccess) return -1;
  *name = "tc_prefill";
  return 1;
}

}  // namespace bsra
