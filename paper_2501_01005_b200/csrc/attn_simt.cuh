// attn_simt.cuh — persistent CUDA-core paged attention (the paper's T_q = 1 "CUDA Cores
// template", generalised to any tile): fp32 arithmetic, any dtype, D in {64, 128},
// NONE / CAUSAL / CUSTOM masks. It is the fp32 path (BASELINE configs[0]) and the cross-check
// for the tcgen05 kernels.
//
// One CTA per plan queue (grid = num_ctas). For each work item (request, kv head,
// q tile, kv chunk) the 4 warps take 4 head-fused rows at a time (App. A, P:413-414:
// fused row f <-> token f / g, qo head kvh*g + f % g) and stream the chunk's K/V through a
// double-buffered shared-memory tile of 32 tokens gathered page by page from the BSR indices
// with 16-byte cp.async (§3.2.1). Online softmax in the log2 domain.
// Epilogue: unsplit rows write o / lse directly, split rows write an fp32 partial slot
// (App. D.2).
#pragma once
#include "common.cuh"
#include "merge.cuh"

namespace bsra {

constexpr int kSimtTile = 32;  // tokens per shared-memory tile (= one token per lane)
constexpr int kSimtWarps = 4;

template <typename T, int D>
struct SimtSmem {
  static constexpr int kRowBytes = D * (int)sizeof(T) + 16;  // +16 B pad: conflict-free row reads
  static constexpr int kTileBytes = kSimtTile * kRowBytes;
  static constexpr int kBytes = 2 /*stages*/ * 2 /*K,V*/ * kTileBytes;
};

// TKV = element type of the pools (T, or __nv_fp8_e4m3 for the fp8 KV cache, R28)
template <typename T, int D>
__device__ __forceinline__ void simt_load_tile(const AttnParams& p, uint8_t* sk, uint8_t* sv, int64_t t0, int n,
                                               int64_t page_begin, int kvh) {
  constexpr int kChunks = D * (int)sizeof(T) / 16;  // 16-byte chunks per token row
  using S = SimtSmem<T, D>;
  const T* kp = reinterpret_cast<const T*>(p.k);
  const T* vp = reinterpret_cast<const T*>(p.v);
  for (int c = threadIdx.x; c < n * kChunks; c += blockDim.x) {
    const int tt = c / kChunks, ch = c % kChunks;
    const int64_t t = t0 + tt;
    const int64_t page = p.kv_ragged ? 0 : __ldg(p.page_indices + page_begin + t / p.page_size);
    const int64_t slot = p.kv_ragged ? page_begin + t : t % p.page_size;
    const T* ksrc = kp + page * p.ks0 + slot * p.ks1 + kvh * p.ks2 + ch * (16 / (int)sizeof(T));
    const T* vsrc = vp + page * p.vs0 + slot * p.vs1 + kvh * p.vs2 + ch * (16 / (int)sizeof(T));
    cp_async16(sk + tt * S::kRowBytes + ch * 16, ksrc);
    cp_async16(sv + tt * S::kRowBytes + ch * 16, vsrc);
  }
}

template <typename T, typename TKV, int D>
__global__ void __launch_bounds__(kSimtWarps * 32) attn_simt_kernel(const __grid_constant__ AttnParams p) {
  using S = SimtSmem<TKV, D>;
  constexpr int kPer = D / 32;               // output dims owned per lane
  constexpr int kVecN = Vec<T>::N;           // q elements per 16-byte vector
  constexpr int kVecK = Vec<TKV>::N;         // K elements per 16-byte vector
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sk[2] = {smem, smem + 2 * S::kTileBytes};
  uint8_t* sv[2] = {smem + S::kTileBytes, smem + 3 * S::kTileBytes};

  const PlanView pv = load_plan(p.plan);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.g;
  const int it0 = pv.cta_indptr[blockIdx.x], it1 = pv.cta_indptr[blockIdx.x + 1];

  for (int it = it0; it < it1; ++it) {
    const int req = pv.item_req[it], kvh = pv.item_kvh[it], qt = pv.item_qtile[it];
    const int64_t kb = pv.item_kb[it], ke = pv.item_ke[it];
    const int slot = pv.item_slot[it];
    const int64_t qo_begin = pv.req_qo_begin[req];
    const int lq = pv.req_qo_len[req];
    const int64_t lk = pv.req_kv_len[req];
    const int64_t page_begin = pv.req_page_begin[req];
    const int row0 = qt * pv.T_q;
    const int nrows = min(pv.T_q, lq * g - row0);

    for (int rb = 0; rb < nrows; rb += kSimtWarps) {
      const int r = rb + warp;  // row within the tile
      const bool valid = r < nrows;
      const int f = row0 + (valid ? r : 0);
      const int tok = f / g;
      const int head = kvh * g + f % g;
      const int64_t causal_lim = lk - lq + tok;  // visible iff t <= lim (right aligned)
      const int64_t mbase = p.mask_mode == 2 ? p.mask_indptr[req] + (int64_t)tok * lk : 0;
      const float slope = p.alibi ? alibi_slope_raw(p, head) : 0.f;  // ALiBi (R30)

      // q row in registers (every lane holds all D values for the lane = token dot products)
      float qv[D];
      {
        const T* qsrc = reinterpret_cast<const T*>(p.q) + ((qo_begin + tok) * p.H_qo + head) * (int64_t)D;
#pragma unroll
        for (int c = 0; c < D / kVecN; ++c) {
          uint4 u = valid ? __ldg(reinterpret_cast<const uint4*>(qsrc) + c) : make_uint4(0, 0, 0, 0);
          Vec<T>::to_float(u, qv + c * kVecN);
        }
      }
      if (p.rope) {  // QueryTransform (R31): the row sits at position l_kv - l_qo + tok
#pragma unroll
        for (int i = 0; i < D / 2; ++i) {
          float sn, cs;
          rope_sincos(causal_lim, p.rope_f[i], sn, cs);
          const float x = qv[i], y = qv[i + D / 2];
          qv[i] = to_f<T>(from_float<T>(x * cs - y * sn));  // a query tensor of dtype T
          qv[i + D / 2] = to_f<T>(from_float<T>(y * cs + x * sn));
        }
      }
      float m = -INFINITY, dsum = 0.f;
      float acc[kPer];
#pragma unroll
      for (int j = 0; j < kPer; ++j) acc[j] = 0.f;

      const int ntiles = (int)((ke - kb + kSimtTile - 1) / kSimtTile);
      __syncthreads();  // previous users of the stage buffers are done
      if (ntiles > 0) simt_load_tile<TKV, D>(p, sk[0], sv[0], kb, (int)imin64(kSimtTile, ke - kb), page_begin, kvh);
      cp_async_commit();
      for (int ti = 0; ti < ntiles; ++ti) {
        const int st = ti & 1;
        const int64_t t0 = kb + (int64_t)ti * kSimtTile;
        const int n = (int)imin64(kSimtTile, ke - t0);
        if (ti + 1 < ntiles) {
          const int64_t t1 = t0 + kSimtTile;
          simt_load_tile<TKV, D>(p, sk[st ^ 1], sv[st ^ 1], t1, (int)imin64(kSimtTile, ke - t1), page_begin, kvh);
        }
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();

        // ---- scores: lane = token
        const int64_t t = t0 + lane;
        bool vis = valid && lane < n;
        if (vis && p.mask_mode == 1) vis = t <= causal_lim;
        if (vis && p.mask_mode == 2) vis = mask_bit(p.mask, mbase + t);
        if (vis && p.window > 0) vis = t >= causal_lim - p.window + 1;  // sliding window (R26)
        float s = -INFINITY;
        if (vis) {
          const uint4* krow = reinterpret_cast<const uint4*>(sk[st] + lane * S::kRowBytes);
          float dot = 0.f;
          if (p.rope) {  // KeyTransform (R31): key t at position t, rotated then rounded to T
            const TKV* kr = reinterpret_cast<const TKV*>(krow);
#pragma unroll
            for (int i = 0; i < D / 2; ++i) {
              float sn, cs;
              rope_sincos(t, p.rope_f[i], sn, cs);
              const float x = to_f<TKV>(kr[i]), y = to_f<TKV>(kr[i + D / 2]);
              dot = fmaf(qv[i], to_f<T>(from_float<T>(x * cs - y * sn)), dot);
              dot = fmaf(qv[i + D / 2], to_f<T>(from_float<T>(y * cs + x * sn)), dot);
            }
          } else {
#pragma unroll
            for (int c = 0; c < D / kVecK; ++c) {
              float kf[kVecK];
              Vec<TKV>::to_float(krow[c], kf);
#pragma unroll
              for (int e = 0; e < kVecK; ++e) dot = fmaf(qv[c * kVecK + e], kf[e], dot);
            }
          }
          float sr = p.soft_cap > 0.f ? soft_cap_raw(p, dot) : dot;  // soft-cap (R27)
          if (p.alibi) sr += slope * (float)(t - causal_lim);         // ALiBi (R30): t - p
          s = sr * p.scale_log2;
        }
        const float mt = warp_max(s);
        const float mnew = fmaxf(m, mt);
        if (mnew != -INFINITY) {
          const float alpha = exp2f(m - mnew);  // m = -inf -> 0
          const float pr = vis ? exp2f(s - mnew) : 0.f;
          dsum = dsum * alpha + warp_sum(pr);
#pragma unroll
          for (int j = 0; j < kPer; ++j) acc[j] *= alpha;
          m = mnew;
          // ---- O += P V: lane owns dims [lane*kPer, lane*kPer + kPer)
          for (int tt = 0; tt < n; ++tt) {
            const float pt = __shfl_sync(0xffffffffu, pr, tt);
            const TKV* vrow = reinterpret_cast<const TKV*>(sv[st] + tt * S::kRowBytes) + lane * kPer;
#pragma unroll
            for (int j = 0; j < kPer; ++j) acc[j] = fmaf(pt, to_f<TKV>(vrow[j]), acc[j]);
          }
        }
        __syncthreads();  // stage st is free for the load issued in the next iteration
      }
      cp_async_wait<0>();

      // ---- epilogue
      if (valid) {
        const bool empty = dsum == 0.f;
        const float inv = empty ? 0.f : p.v_scale / dsum;  // v_scale: fp8 KV (R28), else 1
        const float lse = empty ? -INFINITY : (m + __log2f(dsum)) * kLn2;
        if (slot < 0) {
          const int64_t orow = (qo_begin + tok) * p.H_qo + head;
          if (p.o_f32) {
            float* o = reinterpret_cast<float*>(p.o) + orow * D + lane * kPer;
#pragma unroll
            for (int j = 0; j < kPer; ++j) o[j] = acc[j] * inv;
          } else {
            T* o = reinterpret_cast<T*>(p.o) + orow * D + lane * kPer;
#pragma unroll
            for (int j = 0; j < kPer; ++j) o[j] = from_float<T>(acc[j] * inv);
          }
          if (p.lse && lane == 0) p.lse[orow] = lse;
        } else {
          const int64_t prow = (int64_t)slot * p.T_slot + r;
          float* po = p.part_o + prow * D + lane * kPer;
#pragma unroll
          for (int j = 0; j < kPer; ++j) po[j] = acc[j] * inv;
          if (lane == 0) p.part_lse[prow] = lse;
        }
      }
    }
    if (slot >= 0 && p.fused_merge) {  // split item: the CTA completing its merge list folds it
      __shared__ int s_flag;
      fused_contraction<T, D>(p, pv, slot, threadIdx.x, blockDim.x, 0, &s_flag);
    }
  }
}

}  // namespace bsra
