// tc_kernels.cu — host side of the tcgen05 kernels: TMA tensor maps over q and the paged K/V
// pools (built per run(); a captured graph bakes them) and the launch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tc_decode.cuh"
#include "tc_decode_f8.cuh"
#include "tc_kernels.hpp"
#include "tc_prefill.cuh"

namespace bsra {
namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

// q [N, H_qo, 128] contiguous: dims (d, head, token), box (64, hb, tb), 128B swizzle
bool make_q_map(CUtensorMap* m, const void* q, bool f16, int H_qo, int64_t N, int hb, int tb, int D = 128) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)H_qo, (cuuint64_t)std::max<int64_t>(N, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)H_qo * D * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)hb, (cuuint32_t)tb};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q),
             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// paged pool: element (page, slot, head, d) at page*s0 + slot*s1 + head*s2 + d (elements).
// 4-D view ordered (d, head, slot, page) — coordinates in that order — box (64, 1, B, 1).
// Contiguous KV uses the same view with slot = token (extent N, clipped there) and one page.
// f8: E4M3 pools (1-byte elements), box (128, 1, B, 1) = one 128-byte row per token.
bool make_pool_map(CUtensorMap* m, const void* pool, bool f16, int H_kv, int64_t page_size, int64_t s0, int64_t s1,
                   int64_t s2, int B, int64_t npages = 0x7fffffff, bool f8 = false, int D = 128) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t es_b = f8 ? 1 : 2;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)H_kv, (cuuint64_t)std::max<int64_t>(page_size, 1), (cuuint64_t)npages};
  cuuint64_t strides[3] = {(cuuint64_t)s2 * es_b, (cuuint64_t)s1 * es_b, (cuuint64_t)s0 * es_b};
  cuuint32_t box[4] = {f8 ? 128u : 64u, 1, (cuuint32_t)B, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  const CUtensorMapDataType dt =
      f8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  return enc(m, dt, 4, const_cast<void*>(pool),
             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// paged pool as the 5-D view of the group-major decode tiles (tc_decode kGrp): dims (d_lo 64,
// token_lo 8, half 2, token_hi page_size/8, c = page * cs + head), strides (-, s1, 64, 8 s1, s2)
// elements with cs = s0 / s2 (so c * s2 = page * s0 + head * s2); box (64, 8, 2, B/8, 1) lands as
// [B/8 groups][half][8 rows][128 B] — a whole page (both halves) per box. Needs s0 % s2 == 0 and
// page_size % 8 == 0; the caller falls back to the 4-D map otherwise.
bool make_pool_map5(CUtensorMap* m, const void* pool, bool f16, int64_t page_size, int64_t s0, int64_t s1, int64_t s2,
                    int B, int* cs_out) {
  auto enc = get_encode();
  if (!enc || s2 <= 0 || s0 % s2 || page_size % 8 || B % 8) return false;
  const int64_t cs = s0 / s2;
  if (cs <= 0 || cs > (1 << 20)) return false;
  cuuint64_t dims[5] = {64, 8, 2, (cuuint64_t)(page_size / 8), 0x7fffffffull};  // 2^32 - 1 encodes but traps at run time
  cuuint64_t strides[4] = {(cuuint64_t)s1 * 2, 128, (cuuint64_t)s1 * 16, (cuuint64_t)s2 * 2};
  cuuint32_t box[5] = {64, 8, 2, (cuuint32_t)(B / 8), 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  *cs_out = (int)cs;
  return enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(pool),
             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// pool as a 2-D tensor [rows, 128] (a row = one (page, slot, head) of D = 128 contiguous elements)
// for TMA gather4: box {64 columns, 1 row}, 128B swizzle; 4 rows per instruction
bool make_row_map(CUtensorMap* m, const void* pool, bool f16) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {128, 0x7fffffffull};
  cuuint64_t strides[1] = {128 * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  return enc(m, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool),
             dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int kC, int kMask, bool kF8, bool kRope = false, bool kRow = false, int kD = 128, bool kGrp = false>
cudaError_t launch_decode_t(const TcParams& tp, int grid, cudaStream_t st) {
  static bool attr = false;
  if constexpr (kF8) {  // fp8 KV cache: K in TMEM, converter warps (tc_decode_f8.cuh)
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(tc_decode_f8_kernel<kC, kMask, false>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, f8d::kSmemBytes);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(tc_decode_f8_kernel<kC, kMask, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               f8d::kSmemBytes);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    if (tp.f16) return launch_tc(tc_decode_f8_kernel<kC, kMask, true>, grid, f8d::threads_for(kC), f8d::kSmemBytes, st, tp);
    return launch_tc(tc_decode_f8_kernel<kC, kMask, false>, grid, f8d::threads_for(kC), f8d::kSmemBytes, st, tp);
  } else {
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tc_decode_kernel<kC, kMask, false, kRope, kRow, kD, kGrp>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, dec::kSmemBytes);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(tc_decode_kernel<kC, kMask, true, kRope, kRow, kD, kGrp>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, dec::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int nt = dec::threads_for(kRope, kRow);
  if (tp.f16) return launch_tc(tc_decode_kernel<kC, kMask, true, kRope, kRow, kD, kGrp>, grid, nt, dec::kSmemBytes, st, tp);
  return launch_tc(tc_decode_kernel<kC, kMask, false, kRope, kRow, kD, kGrp>, grid, nt, dec::kSmemBytes, st, tp);
  }
}

template <int kC, bool kF8>
cudaError_t launch_decode_m(int mask, const TcParams& tp, int grid, cudaStream_t st) {
  if constexpr (!kF8) {
    if (tp.p.D == 64) {  // head_dim 64 (box gather only)
      switch (mask) {
        case 0: return launch_decode_t<kC, 0, false, false, false, 64>(tp, grid, st);
        case 1: return launch_decode_t<kC, 1, false, false, false, 64>(tp, grid, st);
        default: return launch_decode_t<kC, 2, false, false, false, 64>(tp, grid, st);
      }
    }
    if (tp.cp) {  // row gather variant (page sizes TMA boxes cannot tile)
      switch (mask) {
        case 0: return launch_decode_t<kC, 0, false, false, true>(tp, grid, st);
        case 1: return launch_decode_t<kC, 1, false, false, true>(tp, grid, st);
        default: return launch_decode_t<kC, 2, false, false, true>(tp, grid, st);
      }
    }
    if (tp.p.rope) {  // fused RoPE variant (R31)
      switch (mask) {
        case 0: return launch_decode_t<kC, 0, false, true>(tp, grid, st);
        case 1: return launch_decode_t<kC, 1, false, true>(tp, grid, st);
        default: return launch_decode_t<kC, 2, false, true>(tp, grid, st);
      }
    }
    if (tp.grp) {  // group-major tiles: one 5-D box per page (paged pools)
      switch (mask) {
        case 0: return launch_decode_t<kC, 0, false, false, false, 128, true>(tp, grid, st);
        case 1: return launch_decode_t<kC, 1, false, false, false, 128, true>(tp, grid, st);
        default: return launch_decode_t<kC, 2, false, false, false, 128, true>(tp, grid, st);
      }
    }
  }
  switch (mask) {
    case 0: return launch_decode_t<kC, 0, kF8>(tp, grid, st);
    case 1: return launch_decode_t<kC, 1, kF8>(tp, grid, st);
    default: return launch_decode_t<kC, 2, kF8>(tp, grid, st);
  }
}

template <bool kF8>
cudaError_t launch_decode_f(int kc, int mask, const TcParams& tp, int grid, cudaStream_t st) {
  switch (kc) {
    case 4: return launch_decode_m<4, kF8>(mask, tp, grid, st);
    case 8: return launch_decode_m<8, kF8>(mask, tp, grid, st);
    default: return launch_decode_m<16, kF8>(mask, tp, grid, st);
  }
}

cudaError_t launch_decode(bool f8, int kc, int mask, const TcParams& tp, int grid, cudaStream_t st) {
  return f8 ? launch_decode_f<true>(kc, mask, tp, grid, st) : launch_decode_f<false>(kc, mask, tp, grid, st);
}

}  // namespace

bool make_q_map_ext(CUtensorMap* m, const void* q, bool f16, int H_qo, int64_t N, int hb, int tb) {
  return make_q_map(m, q, f16, H_qo, N, hb, tb);
}
// Group-major K/V tiles (one 5-D box per page, tp.grp = 1) where the pool strides allow it:
// paged 16-bit pools with head_dim 128 (not for contiguous KV, fp8 or RoPE launches; A/B builds
// with -DBSRA_NO_GRP keep the half-major 4-D boxes). Returns false (tp untouched) otherwise.
bool make_kv_maps5(TcParams& tp, const AttnParams& p, const TcLaunch& L, int B) {
#ifdef BSRA_NO_GRP
  return false;
#endif
  if (L.ragged || L.f8kv || L.rope || p.D != 128) return false;
  int cs_k = 0, cs_v = 0;
  if (!make_pool_map5(&tp.tk, p.k, L.f16, L.page_size, p.ks0, p.ks1, p.ks2, B, &cs_k) ||
      !make_pool_map5(&tp.tv, p.v, L.f16, L.page_size, p.vs0, p.vs1, p.vs2, B, &cs_v) || cs_k != cs_v)
    return false;
  tp.grp = 1;
  tp.cs = cs_k;
  return true;
}

// K and V maps for a launch: paged pools, or contiguous KV (token extent L.total_kv, one page)
bool make_kv_maps(TcParams& tp, const AttnParams& p, const TcLaunch& L, int B) {
  if (L.ragged)
    return make_pool_map(&tp.tk, p.k, L.f16, p.H_kv, L.total_kv, p.ks1, p.ks1, p.ks2, B, 1, L.f8kv, p.D) &&
           make_pool_map(&tp.tv, p.v, L.f16, p.H_kv, L.total_kv, p.vs1, p.vs1, p.vs2, B, 1, L.f8kv, p.D);
  return make_pool_map(&tp.tk, p.k, L.f16, p.H_kv, L.page_size, p.ks0, p.ks1, p.ks2, B, 0x7fffffff, L.f8kv, p.D) &&
         make_pool_map(&tp.tv, p.v, L.f16, p.H_kv, L.page_size, p.vs0, p.vs1, p.vs2, B, 0x7fffffff, L.f8kv, p.D);
}

int tc_launch(const AttnParams& p, const TcLaunch& L, cudaStream_t st, const char** name, const char** why) {
  *why = "";
  if (p.D != 128 && !(p.D == 64 && L.T_q == 16 && !L.f8kv && !L.rope)) {
    *why = "head_dim 64 runs on tensor cores only for bf16/f16 decode tiles without RoPE";
    return 0;
  }
  const int g = p.g;
  if (!is_pow2(g)) { *why = "group size not a power of two"; return 0; }
  const int ps = L.page_size;
  // contiguous KV: any tile start is one 128-token box at a token coordinate
  const int B = L.ragged ? 128 : std::min(ps, 128);
  // pages a TMA box cannot tile (B_c < 8, or B_c neither dividing nor a multiple of 128): decode
  // tiles gather rows with 16-byte cp.async instead (any page size, any chunk alignment)
  const bool box_ok = L.ragged || (ps >= 8 && (128 % ps == 0 || ps % 128 == 0) && L.align % B == 0);
  const bool cp_gather = L.T_q == 16 && !L.f8kv && !L.rope && p.D == 128 && (!box_ok || L.force_cp);
  // row gather flavour: TMA gather4 when K and V share strides that are whole D-element rows (the
  // NHD / HND pools), else 16-byte cp.async
  const bool rows_ok = !L.ragged && p.ks0 == p.vs0 && p.ks1 == p.vs1 && p.ks2 == p.vs2 && p.ks0 % 128 == 0 &&
                       p.ks1 % 128 == 0 && p.ks2 % 128 == 0;
  if (!box_ok && !cp_gather) {
    *why = "page size must divide 128 (>= 8) or be a multiple of 128 (prefill / fp8 / RoPE tiles)";
    return 0;
  }
  if (L.T_q == 16) {
    TcParams tp;
    std::memset(&tp, 0, sizeof(tp));
    tp.p = p;
    tp.box_tok = B;
    tp.q_hb = g <= 16 ? g : 16;
    tp.q_tb = g <= 16 ? 16 / g : 1;
    tp.f16 = L.f16;
    tp.pdl = L.pdl;
    tp.cp = cp_gather ? (rows_ok && !L.force_cp_async ? 2 : 1) : 0;
    bool maps_ok = make_q_map(&tp.tq, p.q, L.f16, p.H_qo, L.total_qo, tp.q_hb, tp.q_tb, p.D);
    // group-major tiles (one box per page) where the pool strides allow the 5-D view
    if (tp.cp == 0 && !make_kv_maps5(tp, p, L, B)) maps_ok = maps_ok && make_kv_maps(tp, p, L, B);
    if (tp.cp == 2) {
      tp.row_s0 = p.ks0 / 128;
      tp.row_s1 = p.ks1 / 128;
      tp.row_s2 = p.ks2 / 128;
      maps_ok = maps_ok && make_row_map(&tp.tk, p.k, L.f16) && make_row_map(&tp.tv, p.v, L.f16);
    }
    if (!maps_ok) {
      *why = "cuTensorMapEncodeTiled failed";
      return -1;
    }
    if (launch_decode(L.f8kv, L.kc, L.mask, tp, L.grid, st) != cudaSuccess) return -1;
    *name = "tc_decode";
    return 1;
  }
  if (L.f8kv) { *why = "fp8 KV with T_q > 16 runs on the CUDA-core kernel"; return 0; }
  if (L.rope) { *why = "fused RoPE with T_q > 16 runs on the CUDA-core kernel"; return 0; }
  if (L.T_q == 64 || L.T_q == 128 || L.T_q == 256) {
    return tc_prefill_launch(p, L, st, name, why, B);
  }
  *why = "no tcgen05 kernel for this tile";
  return 0;
}

}  // namespace bsra
