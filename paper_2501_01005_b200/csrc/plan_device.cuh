// plan_device.cuh — Algorithm 1 on the device (the paper's future work: "move the
// scheduler to device"). One CTA of 1024 threads turns the DEVICE BSR arrays of a step into the
// same int32 plan image the host scheduler (scheduler.cpp) builds, bit for bit, so a step's
// inspector can be captured in a CUDA graph together with its run() calls.
//
// Steps and readings are those of scheduler.cpp (R11-R17): lengths from the BSR
// arrays (a1); rows = (request, kv head, q tile) with the causal-effective / windowed range
// (R12, R13, R26); L = ceil(sum / #CTA) floored at L_min and 1, rounded up to the alignment
// (R11); fixed-stride chunks, one empty chunk for an empty row (R14); sort by (descending
// length, ascending work index) — a bitonic sort of (0x7fffffff - len, w) keys, unique, so the
// order is the host's (R15); greedy min-(cost, cta) assignment — one warp keeps the
// per-CTA costs and takes the arg-min of packed (cost, cta) keys per item; writethrough and merge
// lists per split row (R17). The T_q tile is fixed by the engine (cfg.tile_q).
//
// Errors (malformed arrays, bounds) leave an empty plan (n_items = 0, so run() launches find no
// work) and a nonzero code in header word 12 (bsra_plan_device_status reads it back).
#pragma once
#include <cstdint>

namespace bsra {

struct DevPlanParams {
  const int32_t* qo_indptr;       // [batch+1] device
  const int32_t* kv_page_indptr;  // [batch+1] device
  const int32_t* kv_last_page_len;  // [batch] device
  int32_t* image;                 // workspace plan section
  int32_t* scratch;               // workspace device-planner scratch section
  int64_t scratch_words;
  int32_t cap_words;              // plan section capacity
  int32_t batch, H_kv, g, page_size, mask, num_ctas, T_q, align, L_min, window, max_total_qo_rows;
  int64_t alpha, beta;
};

namespace devplan {
constexpr int kThreads = 1024;
constexpr int kMaxSort = 16384;  // items sorted in shared memory (128 KB of keys)
constexpr int kSmemBytes = kMaxSort * 8 + (kThreads + 1) * 8 + 64;  // sort keys + scan scratch
enum : int32_t { kOk = 0, kEMalformed = 1, kEBounds = 2, kETooLarge = 3 };
}  // namespace devplan

__device__ __forceinline__ int64_t dp_cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// exclusive prefix sum of a[0..n) in place (global or shared memory), returns the total
__device__ int64_t dp_block_scan(int32_t* a, int32_t n, int64_t* sh) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int64_t s = 0;
  for (int i = lo; i < hi; ++i) s += a[i];
  sh[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t run = 0;
    for (int k = 0; k < nt; ++k) {
      const int64_t v = sh[k];
      sh[k] = run;
      run += v;
    }
    sh[nt] = run;
  }
  __syncthreads();
  int64_t run = sh[tid];
  for (int i = lo; i < hi; ++i) {
    const int32_t v = a[i];
    a[i] = (int32_t)run;
    run += v;
  }
  const int64_t total = sh[nt];
  __syncthreads();
  return total;
}

__device__ __forceinline__ void dp_fail(const DevPlanParams& P, int32_t code) {
  if (threadIdx.x == 0) {
    int32_t* im = P.image;
    im[0] = 0x41525342;
    im[1] = 1;
    im[2] = P.num_ctas;
    im[3] = P.T_q;
    im[4] = 1;
    for (int k = 5; k < 16; ++k) im[k] = 0;
    im[8] = 0;  // batch 0: nothing to do
    im[9] = P.g;
    im[10] = P.H_kv;
    im[11] = P.mask;
    im[12] = code;
    for (int c = 0; c <= P.num_ctas; ++c) im[16 + c] = 0;  // empty queues
  }
}

__global__ void __launch_bounds__(devplan::kThreads, 1) plan_device_kernel(const DevPlanParams P) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem);                       // [kMaxSort]
  int64_t* sh = reinterpret_cast<int64_t*>(smem + devplan::kMaxSort * 8);   // [kThreads + 1] scan / misc
  __shared__ int32_t s_err, s_R, s_N, s_nlists, s_nslots;
  __shared__ int64_t s_total, s_L;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int B = P.batch, H = P.H_kv, g = P.g, T = P.T_q;
  if (tid == 0) s_err = 0;
  __syncthreads();
  // scratch layout (int32): qo[B] kv[B] rowoff[B+1] | per row: rb[R] re[R] rn[R] rfirst[R] rslot[R]
  //                         | per chunk: cta[N] pos[N] | cnt[num_ctas+1]
  int32_t* qo = P.scratch;
  int32_t* kv = qo + B;
  int32_t* rowoff = kv + B;
  // ---- a1: lengths and validation
  for (int i = tid; i < B; i += nt) {
    const int32_t q0 = P.qo_indptr[i], q1 = P.qo_indptr[i + 1];
    const int32_t p0 = P.kv_page_indptr[i], p1 = P.kv_page_indptr[i + 1];
    const int64_t lq = (int64_t)q1 - q0, n = (int64_t)p1 - p0;
    int64_t lk = 0;
    bool bad = lq < 0 || n < 0 || (i == 0 && (q0 != 0 || p0 != 0));
    if (n > 0) {
      const int32_t last = P.kv_last_page_len[i];
      bad = bad || last < 1 || last > P.page_size;
      lk = (n - 1) * (int64_t)P.page_size + last;
    }
    bad = bad || lk > 0x7fffffff;
    if (bad) atomicMax(&s_err, devplan::kEMalformed);
    qo[i] = (int32_t)lq;
    kv[i] = (int32_t)lk;
    rowoff[i] = bad ? 0 : (int32_t)(H * dp_cdiv(lq * g, T));
  }
  __syncthreads();
  if (s_err) {
    dp_fail(P, s_err);
    return;
  }
  if (B > 0 && tid == 0 && (int64_t)P.qo_indptr[B] > P.max_total_qo_rows) s_err = devplan::kEBounds;
  const int64_t R64 = dp_block_scan(rowoff, B, sh);
  if (tid == 0) rowoff[B] = (int32_t)R64;
  if (s_err || R64 > devplan::kMaxSort || 2 * (int64_t)B + 1 + 5 * R64 > P.scratch_words) {
    dp_fail(P, s_err ? s_err : devplan::kETooLarge);
    return;
  }
  const int32_t R = (int32_t)R64;
  int32_t* rb = rowoff + B + 1;
  int32_t* re = rb + R;
  int32_t* rn = re + R;
  int32_t* rfirst = rn + R;
  int32_t* rslot = rfirst + R;
  // ---- rows (request, kv head, q tile) and their KV ranges [b, e)
  int64_t part = 0;
  for (int r = tid; r < R; r += nt) {
    int lo = 0, hi = B;  // request i: rowoff[i] <= r < rowoff[i+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rowoff[mid] <= r) lo = mid;
      else hi = mid;
    }
    const int i = lo;
    const int64_t lq = qo[i], lk = kv[i];
    const int64_t fused = lq * g;
    const int64_t ntile = dp_cdiv(fused, T);
    const int64_t local = r - rowoff[i];
    const int64_t t = local % ntile;
    int64_t e = lk;
    if (P.mask == 1) {
      const int64_t hi2 = min((t + 1) * T, fused);
      const int64_t last_tok = dp_cdiv(hi2, g) - 1;
      e = min(max(lk - lq + last_tok + 1, (int64_t)0), lk);
    }
    int64_t b = 0;
    if (P.window > 0) {
      const int64_t first_tok = (t * T) / g;
      b = max((int64_t)0, lk - lq + first_tok - P.window + 1);
      const int64_t al = max(1, P.align);
      b = min(b / al * al, e);
    }
    rb[r] = (int32_t)b;
    re[r] = (int32_t)e;
    part += e - b;
  }
  sh[tid] = part;
  __syncthreads();
  if (tid == 0) {
    int64_t tot = 0;
    for (int k = 0; k < nt; ++k) tot += sh[k];
    int64_t L = max(max(dp_cdiv(tot, P.num_ctas), (int64_t)P.L_min), (int64_t)1);
    const int64_t al = max(1, P.align);
    L = dp_cdiv(L, al) * al;
    s_total = tot;
    s_L = L;
    if (L > 0x7fffffff) s_err = devplan::kETooLarge;
  }
  __syncthreads();
  if (s_err) {
    dp_fail(P, s_err);
    return;
  }
  const int64_t L = s_L;
  // ---- chunks per row; split rows get consecutive slots (in row order, R17)
  for (int r = tid; r < R; r += nt) {
    const int64_t n = max((int64_t)1, dp_cdiv((int64_t)re[r] - rb[r], L));
    rn[r] = (int32_t)n;
    rfirst[r] = (int32_t)n;
    rslot[r] = n > 1 ? (int32_t)n : 0;
  }
  __syncthreads();
  const int64_t N64 = dp_block_scan(rfirst, R, sh);
  const int64_t NS64 = dp_block_scan(rslot, R, sh);
  if (N64 > devplan::kMaxSort) {
    dp_fail(P, devplan::kETooLarge);
    return;
  }
  const int32_t N = (int32_t)N64, NS = (int32_t)NS64;
  // lists = split rows
  int32_t nlist_part = 0;
  for (int r = tid; r < R; r += nt) nlist_part += rn[r] > 1;
  sh[tid] = nlist_part;
  __syncthreads();
  if (tid == 0) {
    int64_t tot = 0;
    for (int k = 0; k < nt; ++k) tot += sh[k];
    s_nlists = (int32_t)tot;
    s_N = N;
    s_nslots = NS;
  }
  __syncthreads();
  const int32_t NL = s_nlists;
  const int64_t words = 16 + (P.num_ctas + 1) + 6 * (int64_t)N + (NL + 1) + NS + 3 * (int64_t)NL + 4 * (int64_t)B;
  int32_t* cta_of = rslot + R;
  int32_t* pos_of = cta_of + N;
  int32_t* cnt = pos_of + N;
  if (words > P.cap_words || (int64_t)(cnt + P.num_ctas + 1 - P.scratch) > P.scratch_words) {
    dp_fail(P, devplan::kETooLarge);
    return;
  }
  // ---- sort keys: (0x7fffffff - len) << 32 | w, ascending = (descending length, ascending w)
  int sortn = 1;
  while (sortn < N) sortn <<= 1;
  for (int r = tid; r < R; r += nt) {
    const int32_t f = rfirst[r], n = rn[r];
    const int64_t b = rb[r], e = re[r];
    for (int j = 0; j < n; ++j) {
      const int64_t cb = b + (int64_t)j * L, ce = min(b + (int64_t)(j + 1) * L, e);
      keys[f + j] = ((uint64_t)(0x7fffffff - (ce - cb)) << 32) | (uint32_t)(f + j);
    }
  }
  for (int k = N + tid; k < sortn; k += nt) keys[k] = ~0ull;  // padding sorts last
  __syncthreads();
  for (int size = 2; size <= sortn; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int k = tid; k < sortn; k += nt) {
        const int o = k ^ stride;
        if (o > k) {
          const bool up = (k & size) == 0;
          const uint64_t a = keys[k], c = keys[o];
          if ((a > c) == up) {
            keys[k] = c;
            keys[o] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  // ---- greedy: one warp; lane l holds the costs of CTAs l, l+32, ...; per item the arg-min of
  // packed (cost << 12 | cta) keys (ties -> lower cta id), then cost += alpha*T_q + beta*len
  if (tid < 32) {
    constexpr int kMaxPer = 16;  // num_ctas <= 512
    uint64_t cost[kMaxPer];
    int32_t mycnt[kMaxPer];
#pragma unroll
    for (int k = 0; k < kMaxPer; ++k) {
      cost[k] = 0;
      mycnt[k] = 0;
    }
    const int nc = P.num_ctas;
    for (int k = 0; k < N; ++k) {
      const uint64_t key = keys[k];
      const int32_t w = (int32_t)(key & 0xffffffffu);
      const int64_t len = 0x7fffffff - (int64_t)(key >> 32);
      uint64_t best = ~0ull;
#pragma unroll
      for (int q = 0; q < kMaxPer; ++q) {
        const int c = tid + 32 * q;
        if (c < nc) {
          const uint64_t kk = (cost[q] << 12) | (uint64_t)c;
          best = kk < best ? kk : best;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
      }
      const int c = (int)(best & 0xfff);
      if ((c & 31) == tid) {
        const int q = c >> 5;
#pragma unroll
        for (int qq = 0; qq < kMaxPer; ++qq)
          if (qq == q) {
            cta_of[w] = c;
            pos_of[w] = mycnt[qq]++;
            cost[qq] += (uint64_t)(P.alpha * T + P.beta * len);
          }
      }
    }
#pragma unroll
    for (int q = 0; q < kMaxPer; ++q) {
      const int c = tid + 32 * q;
      if (c < nc) cnt[c] = mycnt[q];
    }
  }
  __syncthreads();
  const int64_t n_check = dp_block_scan(cnt, P.num_ctas, sh);  // cnt -> cta_indptr
  if (tid == 0) cnt[P.num_ctas] = (int32_t)n_check;
  __syncthreads();
  // ---- serialise (layout of scheduler.cpp / oracle scheduler_ref.encode_image)
  int32_t* im = P.image;
  int32_t* ind = im + 16;
  int32_t* it_req = ind + P.num_ctas + 1;
  int32_t* it_kvh = it_req + N;
  int32_t* it_qt = it_kvh + N;
  int32_t* it_kb = it_qt + N;
  int32_t* it_ke = it_kb + N;
  int32_t* it_slot = it_ke + N;
  int32_t* l_ind = it_slot + N;
  int32_t* l_slot = l_ind + NL + 1;
  int32_t* l_req = l_slot + NS;
  int32_t* l_kvh = l_req + NL;
  int32_t* l_qt = l_kvh + NL;
  int32_t* q_begin = l_qt + NL;
  int32_t* q_len = q_begin + B;
  int32_t* k_len = q_len + B;
  int32_t* p_begin = k_len + B;
  for (int c = tid; c <= P.num_ctas; c += nt) ind[c] = cnt[c];
  // items, and for split rows the lists (list index = split rows before it, slot base = rslot)
  for (int r = tid; r < R; r += nt) {
    int lo = 0, hi = B;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (rowoff[mid] <= r) lo = mid;
      else hi = mid;
    }
    const int i = lo;
    const int64_t ntile = dp_cdiv((int64_t)qo[i] * g, T);
    const int64_t local = r - rowoff[i];
    const int32_t h = (int32_t)(local / ntile), t = (int32_t)(local % ntile);
    const int32_t f = rfirst[r], n = rn[r];
    const int64_t b = rb[r], e = re[r];
    for (int j = 0; j < n; ++j) {
      const int w = f + j;
      const int32_t at = cnt[cta_of[w]] + pos_of[w];
      it_req[at] = i;
      it_kvh[at] = h;
      it_qt[at] = t;
      it_kb[at] = (int32_t)(b + (int64_t)j * L);
      it_ke[at] = (int32_t)min(b + (int64_t)(j + 1) * L, e);
      it_slot[at] = n > 1 ? rslot[r] + j : -1;
    }
  }
  __syncthreads();
  if (tid == 0) {  // merge lists in row order (R17); few rows are split, a serial walk is enough
    int32_t li = 0;
    l_ind[0] = 0;
    for (int r = 0; r < R; ++r) {
      const int32_t n = rn[r];
      if (n <= 1) continue;
      int lo = 0, hi = B;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (rowoff[mid] <= r) lo = mid;
        else hi = mid;
      }
      const int64_t ntile = dp_cdiv((int64_t)qo[lo] * g, T);
      const int64_t local = r - rowoff[lo];
      for (int j = 0; j < n; ++j) l_slot[rslot[r] + j] = rslot[r] + j;
      l_req[li] = lo;
      l_kvh[li] = (int32_t)(local / ntile);
      l_qt[li] = (int32_t)(local % ntile);
      ++li;
      l_ind[li] = rslot[r] + n;
    }
  }
  for (int i = tid; i < B; i += nt) {
    q_begin[i] = P.qo_indptr[i];
    q_len[i] = qo[i];
    k_len[i] = kv[i];
    p_begin[i] = P.kv_page_indptr[i];
  }
  if (tid == 0) {
    im[0] = 0x41525342;
    im[1] = 1;
    im[2] = P.num_ctas;
    im[3] = T;
    im[4] = (int32_t)L;
    im[5] = N;
    im[6] = NL;
    im[7] = NS;
    im[8] = B;
    im[9] = g;
    im[10] = H;
    im[11] = P.mask;
    im[12] = 0;
    im[13] = 0;
    im[14] = 0;
    im[15] = 0;
  }
}

}  // namespace bsra
