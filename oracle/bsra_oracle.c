/*
 * bsra_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct float64 CPU implementation of paged
 * (block-sparse-row) attention as defined in the FlashInfer paper
 * (arXiv 2501.01005). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no
 * code, header, table or helper with the CUDA path (paper_2501_01005_b200/).
 *
 * What it computes (per request i, query row r, qo head h), two passes, untiled,
 * unsplit, in logical token order:
 *   - Page table = BSR (§3.1.1, fig:focus-sparse-layout):
 *       n_i   = kv_page_indptr[i+1] - kv_page_indptr[i]
 *       l_kv  = n_i == 0 ? 0 : (n_i - 1) * B_c + kv_last_page_len[i]
 *       token t lives in page indices[kv_page_indptr[i] + t / B_c], slot t % B_c
 *   - GQA (§2.1; App. A): kv head = h / g, g = H_qo / H_kv
 *     (reading R5: contiguous head groups).
 *   - Visible set vis(r): NONE: all t; CAUSAL (right aligned, R4):
 *     t <= l_kv - l_qo + r; CUSTOM (R9): bit mask_bit_indptr[i] + r*l_kv + t,
 *     LSB-first in bytes. Masked pairs are skipped, not -inf arithmetic (R10).
 *   - LogitsMask variant, sliding window (§3.2.3; R26): window W > 0
 *     additionally hides t < l_kv - l_qo + r - W + 1 (W keys up to the row's own position).
 *   - LogitsTransform variant, logits soft-cap (R27): cap c > 0 replaces
 *     the scaled logit s by c * tanh(s / c) before Eq. 1-2.
 *   - LogitsTransform variant, ALiBi bias (App. G Table "ALiBi Bias", PAPER.md:554;
 *     DESIGN.md R30): with alibi != 0 the logit of key t for query row r of qo head h becomes
 *     s + slope_h * (t - p), p = l_kv - l_qo + r the row's right-aligned position, applied after
 *     the soft-cap; slope_h from Press et al.: n = 2^floor(log2 H_qo); h < n: 2^(-8(h+1)/n),
 *     else 2^(-4(2(h-n)+1)/n).
 *   - Eq. 1: lse = log sum_{t in vis} exp(s_t), s_t = sm_scale * q.k_t
 *     (R1: the logits are scaled by sm_scale; R2: natural log).
 *   - Eq. 2: o = sum_{t in vis} exp(s_t) / exp(lse) * v_t
 *     (evaluated max-shifted: m = max s_t, Z = sum exp(s_t - m), lse = m + ln Z).
 *   - Empty vis: o = 0, lse = -inf (R3).
 *   - FP8-FP16 mixed precision (App. F): "the query and output remain in
 *     fp16, while the KV-Cache is stored in fp8". K/V may be stored as OCP FP8 E4M3 (kv_dtype 3;
 *     DESIGN.md R28): element value = k_scale * E4M3(byte) (v_scale for V), a per-tensor scale
 *     (1 = the plain format). Nothing else changes: Eq. 1-2 run on the dequantised values.
 *
 * Inputs are the same arrays given to bsra_plan / bsra_run, copied to the host.
 * fp32 / fp16 / bf16 values are upcast exactly to double here (own decoders).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORC_F32 = 0, ORC_F16 = 1, ORC_BF16 = 2, ORC_E4M3 = 3 };
enum { ORC_MASK_NONE = 0, ORC_MASK_CAUSAL = 1, ORC_MASK_CUSTOM = 2 };

/* IEEE binary16 -> double, exact (normal, subnormal, inf, nan). */
static double orc_f16_to_double(uint16_t h) {
  int sign = (h >> 15) & 1;
  int exp = (h >> 10) & 0x1f;
  int man = h & 0x3ff;
  double v;
  if (exp == 0) {
    v = ldexp((double)man, -24); /* subnormal: man * 2^-24 */
  } else if (exp == 31) {
    v = man ? NAN : INFINITY;
  } else {
    v = ldexp((double)(man | 0x400), exp - 25); /* (1.man) * 2^(exp-15) */
  }
  return sign ? -v : v;
}

/* bfloat16 -> double, exact: bf16 is the top half of a binary32. */
static double orc_bf16_to_double(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, sizeof f);
  return (double)f;
}

/* OCP FP8 E4M3 ("E4M3FN") -> double, exact: 1 sign, 4 exponent (bias 7), 3 mantissa bits; no
 * infinities, S.1111.111 is NaN, largest finite 448 (R28). */
static double orc_e4m3_to_double(uint8_t b) {
  int sign = (b >> 7) & 1;
  int exp = (b >> 3) & 0xf;
  int man = b & 0x7;
  double v;
  if (exp == 0) {
    v = ldexp((double)man, -9); /* subnormal: (man / 8) * 2^(1-7) */
  } else if (exp == 15 && man == 7) {
    v = NAN;
  } else {
    v = ldexp((double)(man | 0x8), exp - 10); /* (1.man) * 2^(exp-7) */
  }
  return sign ? -v : v;
}

static double orc_load(const void* base, int dtype, int64_t idx) {
  switch (dtype) {
    case ORC_F32: return (double)((const float*)base)[idx];
    case ORC_F16: return orc_f16_to_double(((const uint16_t*)base)[idx]);
    case ORC_E4M3: return orc_e4m3_to_double(((const uint8_t*)base)[idx]);
    default: return orc_bf16_to_double(((const uint16_t*)base)[idx]);
  }
}

int orc_version(void) { return 1; }

/* RoPE (Su et al., "RoFormer"; the paper's Query/KeyTransform, "fuse ... RoPE"),
 * rotate-half pairing (R31): for i < D/2, theta_i = rope_theta^(-2i/D) / rope_scale and
 * angle a = pos * theta_i (float64, exact positions); the pair (x_i, x_{i+D/2}) becomes
 * (x_i cos a - x_{i+D/2} sin a, x_{i+D/2} cos a + x_i sin a). In place. */
/* Round to the nearest value of a storage dtype (ties to even): ORC_F32 -> float; ORC_F16 /
 * ORC_BF16 -> 11 / 8 significant bits with minimum normal exponent -14 / -126 (subnormals keep
 * that spacing). The plain definition, used for the transformed q / k (R31). */
double orc_round_dtype(double x, int dtype) {
  if (dtype == ORC_F32) return (double)(float)x;
  if (x == 0.0 || !isfinite(x)) return x;
  const int p = dtype == ORC_F16 ? 11 : 8;
  const int emin = dtype == ORC_F16 ? -14 : -126;
  int e;
  frexp(x, &e); /* |x| = m 2^e, 0.5 <= m < 1: leading bit 2^(e-1) */
  int lead = e - 1;
  if (lead < emin) lead = emin;
  const double q = ldexp(1.0, lead - (p - 1)); /* spacing of representable values */
  return nearbyint(x / q) * q;                 /* default rounding mode: to nearest, ties even */
}

void orc_rope_rotate(double* x, int D, double pos, double rope_theta, double rope_scale) {
  const int h = D / 2;
  for (int i = 0; i < h; ++i) {
    const double theta = pow(rope_theta, -2.0 * i / D) / rope_scale;
    const double a = pos * theta;
    const double c = cos(a), sn = sin(a);
    const double x0 = x[i], x1 = x[i + h];
    x[i] = x0 * c - x1 * sn;
    x[i + h] = x1 * c + x0 * sn;
  }
}

/* ALiBi slope of qo head h of H (Press et al. 2022; R30). */
double orc_alibi_slope(int h, int H) {
  int n = 1;
  while (2 * n <= H) n *= 2;
  if (h < n) return pow(2.0, -8.0 * (h + 1) / n);
  return pow(2.0, -4.0 * (2 * (h - n) + 1) / n);
}

/* Exposed for the closed-form pins of the decoders themselves. */
double orc_decode(int dtype, uint32_t bits) {
  if (dtype == ORC_F32) {
    float f;
    memcpy(&f, &bits, sizeof f);
    return (double)f;
  }
  if (dtype == ORC_E4M3) return orc_e4m3_to_double((uint8_t)bits);
  return dtype == ORC_F16 ? orc_f16_to_double((uint16_t)bits) : orc_bf16_to_double((uint16_t)bits);
}

/*
 * orc_paged_attention — returns 0 on success, nonzero on invalid input.
 *   q            [sum l_qo, H_qo, D] contiguous, dtype
 *   k_pool/v_pool element strides {page, token, head}; dim stride 1; kv_dtype (pools' dtype,
 *                ORC_E4M3 for the fp8 KV cache), values scaled by k_scale / v_scale
 *   req_list     optional list of request ids to compute (NULL => all); rows of
 *                other requests in o_out/lse_out are left untouched
 *   o_out        [sum l_qo, H_qo, D] double;  lse_out [sum l_qo, H_qo] double
 */
int orc_paged_attention(int batch, const int32_t* qo_indptr, const int32_t* kv_page_indptr,
                        const int32_t* kv_last_page_len, const int32_t* kv_page_indices,
                        int H_qo, int H_kv, int D, int page_size, int dtype, int kv_dtype,
                        double k_scale, double v_scale, const void* q,
                        const void* k_pool, const void* v_pool, const int64_t* k_strides,
                        const int64_t* v_strides, int mask_mode, const uint8_t* custom_mask,
                        const int64_t* mask_bit_indptr, double sm_scale, int window, double soft_cap, int alibi,
                        double rope_theta, double rope_scale,
                        const int32_t* req_list, int n_req_list, double* o_out, double* lse_out,
                        int num_threads) {
  if (batch < 0 || H_qo <= 0 || H_kv <= 0 || H_qo % H_kv != 0 || D <= 0 || page_size <= 0) return 1;
  if (mask_mode == ORC_MASK_CUSTOM && (!custom_mask || !mask_bit_indptr)) return 2;
  if (rope_theta > 0.0 && (D % 2 != 0 || !(rope_scale > 0.0) || kv_dtype == ORC_E4M3)) return 5;
  const int g = H_qo / H_kv;
  const int nreq = req_list ? n_req_list : batch;

  /* flatten (request, row) work so OpenMP can spread it */
  int64_t nwork = 0;
  for (int a = 0; a < nreq; ++a) {
    int i = req_list ? req_list[a] : a;
    if (i < 0 || i >= batch) return 3;
    nwork += qo_indptr[i + 1] - qo_indptr[i];
  }
  int64_t* work = (int64_t*)malloc(sizeof(int64_t) * 2 * (nwork > 0 ? nwork : 1));
  if (!work) return 4;
  int64_t w = 0;
  for (int a = 0; a < nreq; ++a) {
    int i = req_list ? req_list[a] : a;
    for (int r = 0; r < qo_indptr[i + 1] - qo_indptr[i]; ++r) {
      work[2 * w] = i;
      work[2 * w + 1] = r;
      ++w;
    }
  }
#ifdef _OPENMP
  if (num_threads > 0) omp_set_num_threads(num_threads);
#endif
  int err = 0;
#pragma omp parallel
  {
    double* s = NULL;   /* scores of visible tokens, logical order */
    int32_t* vis = NULL; /* visible token ids */
    int64_t cap = 0;
    double qr[1024], kr[1024]; /* RoPE-rotated q row / k row (D <= 1024) */
#pragma omp for schedule(dynamic, 1)
    for (int64_t wi = 0; wi < nwork; ++wi) {
      const int i = (int)work[2 * wi];
      const int r = (int)work[2 * wi + 1];
      const int l_qo = qo_indptr[i + 1] - qo_indptr[i];
      const int n = kv_page_indptr[i + 1] - kv_page_indptr[i];
      const int64_t l_kv = n == 0 ? 0 : (int64_t)(n - 1) * page_size + kv_last_page_len[i];
      if (l_kv > cap) {
        free(s);
        free(vis);
        cap = l_kv;
        s = (double*)malloc(sizeof(double) * cap);
        vis = (int32_t*)malloc(sizeof(int32_t) * cap);
        if (!s || !vis) {
#pragma omp atomic write
          err = 4;
          cap = 0;
          continue;
        }
      }
      /* visible set, ascending t */
      int64_t nv = 0;
      for (int64_t t = 0; t < l_kv; ++t) {
        int visible = 1;
        if (mask_mode == ORC_MASK_CAUSAL) {
          visible = t <= l_kv - l_qo + r;
        } else if (mask_mode == ORC_MASK_CUSTOM) {
          int64_t j = mask_bit_indptr[i] + (int64_t)r * l_kv + t;
          visible = (custom_mask[j >> 3] >> (j & 7)) & 1;
        }
        if (window > 0 && t < l_kv - l_qo + r - window + 1) visible = 0;
        if (visible) vis[nv++] = (int32_t)t;
      }
      const int64_t row = (int64_t)qo_indptr[i] + r;
      for (int h = 0; h < H_qo; ++h) {
        const int hk = h / g;
        double* o = o_out + (row * H_qo + h) * D;
        if (nv == 0) {
          for (int d = 0; d < D; ++d) o[d] = 0.0;
          lse_out[row * H_qo + h] = -INFINITY;
          continue;
        }
        const int64_t qbase = (row * H_qo + h) * (int64_t)D;
        if (rope_theta > 0.0) { /* QueryTransform: the query row sits at position l_kv - l_qo + r */
          for (int d = 0; d < D; ++d) qr[d] = orc_load(q, dtype, qbase + d);
          orc_rope_rotate(qr, D, (double)(l_kv - l_qo + r), rope_theta, rope_scale);
          /* the transformed query is a query tensor of the input dtype (R31): rounded RN */
          for (int d = 0; d < D; ++d) qr[d] = orc_round_dtype(qr[d], dtype);
        }
        /* pass 1: scores and their max */
        double m = -INFINITY;
        for (int64_t a = 0; a < nv; ++a) {
          const int64_t t = vis[a];
          const int64_t p = kv_page_indices[kv_page_indptr[i] + t / page_size];
          const int64_t kb = p * k_strides[0] + (t % page_size) * k_strides[1] + hk * k_strides[2];
          double dot = 0.0;
          if (rope_theta > 0.0) { /* KeyTransform: key t sits at position t */
            for (int d = 0; d < D; ++d) kr[d] = k_scale * orc_load(k_pool, kv_dtype, kb + d);
            orc_rope_rotate(kr, D, (double)t, rope_theta, rope_scale);
            for (int d = 0; d < D; ++d) kr[d] = orc_round_dtype(kr[d], dtype);
            for (int d = 0; d < D; ++d) dot += qr[d] * kr[d];
          } else
          for (int d = 0; d < D; ++d) dot += orc_load(q, dtype, qbase + d) * (k_scale * orc_load(k_pool, kv_dtype, kb + d));
          s[a] = sm_scale * dot;
          if (soft_cap > 0.0) s[a] = soft_cap * tanh(s[a] / soft_cap);
          if (alibi) s[a] += orc_alibi_slope(h, H_qo) * (double)(t - (l_kv - l_qo + r));
          if (s[a] > m) m = s[a];
        }
        /* pass 2: normaliser, lse, output (Eq. 1-2) */
        double Z = 0.0;
        for (int64_t a = 0; a < nv; ++a) Z += exp(s[a] - m);
        lse_out[row * H_qo + h] = m + log(Z);
        for (int d = 0; d < D; ++d) o[d] = 0.0;
        for (int64_t a = 0; a < nv; ++a) {
          const int64_t t = vis[a];
          const int64_t p = kv_page_indices[kv_page_indptr[i] + t / page_size];
          const int64_t vb = p * v_strides[0] + (t % page_size) * v_strides[1] + hk * v_strides[2];
          const double wgt = exp(s[a] - m) / Z;
          for (int d = 0; d < D; ++d) o[d] += wgt * (v_scale * orc_load(v_pool, kv_dtype, vb + d));
        }
      }
    }
    free(s);
    free(vis);
  }
  free(work);
  return err;
}

/*
 * ⊕ (§2.2), max-shifted form (R3 for the empty state):
 *   m = max(lse_a, lse_b); if m = -inf -> empty (o = 0, lse = -inf)
 *   w_a = e^{lse_a - m}, w_b = e^{lse_b - m}
 *   o = (w_a o_a + w_b o_b) / (w_a + w_b), lse = m + ln(w_a + w_b)
 * rows = number of (row, head) states; each o is D doubles. In-place allowed.
 */
void orc_merge(int64_t rows, int D, const double* o_a, const double* lse_a, const double* o_b,
               const double* lse_b, double* o_out, double* lse_out) {
  for (int64_t x = 0; x < rows; ++x) {
    const double la = lse_a[x], lb = lse_b[x];
    const double m = la > lb ? la : lb;
    if (m == -INFINITY) {
      for (int d = 0; d < D; ++d) o_out[x * D + d] = 0.0;
      lse_out[x] = -INFINITY;
      continue;
    }
    const double wa = exp(la - m), wb = exp(lb - m);
    for (int d = 0; d < D; ++d) o_out[x * D + d] = (wa * o_a[x * D + d] + wb * o_b[x * D + d]) / (wa + wb);
    lse_out[x] = m + log(wa + wb);
  }
}
