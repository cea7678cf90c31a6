// engine.cu — libbsra.so: the C ABI of include/bsra.h.
//
// Engine = the paper's attention wrapper (§3.4): created once with the variant /
// task information (dtype, heads, head_dim, page size, mask) and a caller-owned workspace; plan()
// is the inspector (host Algorithm 1 + H2D of the plan image through pinned staging, App. D
// P:463); run() is the executor (persistent attention kernel + contraction, graph-capturable).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/bsra.h"
#include "attn_simt.cuh"
#include "f8_gather.cuh"
#include "merge.cuh"
#include "plan_device.cuh"
#include "scheduler.hpp"
#include "tc_kernels.hpp"

namespace {

thread_local std::string g_err;

bsra_status fail(bsra_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                         \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess)                                                                     \
      return fail(BSRA_ECUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e));       \
  } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int dtype_size(bsra_dtype t) { return t == BSRA_F32 ? 4 : t == BSRA_E4M3 ? 1 : 2; }

// fp8 KV cache (R28): kv_dtype 0 or == dtype means K/V in dtype
bool kv_is_f8(const bsra_config& c) { return c.kv_dtype == BSRA_E4M3; }
bsra_dtype kv_dtype_of(const bsra_config& c) { return kv_is_f8(c) ? BSRA_E4M3 : c.dtype; }

struct Layout {
  int32_t num_ctas = 0, T_max = 0, T_min = 0;
  size_t plan_words = 0;
  size_t off_plan = 0, off_part_o = 0, off_part_lse = 0, off_counters = 0, off_aux = 0, off_f8 = 0, total = 0;
  size_t off_devscratch = 0, devscratch_words = 0;  // device planner scratch (bsra_plan_device)
  size_t aux_words = 0;  // fp8 prefill gather: src_begin[max_batch+1], kv_off[max_batch+1]
  int64_t f8_rows = 0;   // fp8 prefill gather region: max_total_kv_tokens rows of [H_kv, 128] K and V
};

int tile_mask_of(const bsra_config& c) { return c.tile_set_mask ? c.tile_set_mask : 15; }

bsra_status validate_config(const bsra_config& c) {
  if (c.num_qo_heads <= 0 || c.num_kv_heads <= 0 || c.num_qo_heads % c.num_kv_heads)
    return fail(BSRA_EINVAL, "num_qo_heads must be a positive multiple of num_kv_heads");
  if (c.head_dim != 64 && c.head_dim != 128) return fail(BSRA_EUNSUPPORTED, "head_dim must be 64 or 128");
  if (c.page_size < 1) return fail(BSRA_EINVAL, "page_size < 1");
  if (c.dtype < BSRA_F32 || c.dtype > BSRA_BF16) return fail(BSRA_EINVAL, "bad dtype");
  if (c.o_dtype != c.dtype && c.o_dtype != BSRA_F32) return fail(BSRA_EINVAL, "o_dtype must equal dtype or be F32");
  if (c.mask < BSRA_MASK_NONE || c.mask > BSRA_MASK_CUSTOM) return fail(BSRA_EINVAL, "bad mask");
  if (c.max_batch < 0 || c.max_total_qo_rows < 0) return fail(BSRA_EINVAL, "negative bounds");
  if (c.num_ctas < 0) return fail(BSRA_EINVAL, "num_ctas < 0");
  const int tm = tile_mask_of(c);
  if (tm & ~15) return fail(BSRA_EINVAL, "tile_set_mask has unknown bits");
  if (c.tile_q && c.tile_q != 16 && c.tile_q != 64 && c.tile_q != 128 && c.tile_q != 256)
    return fail(BSRA_EINVAL, "tile_q not in {16,64,128,256}");
  if (c.cost_alpha < 0 || c.cost_beta < 0) return fail(BSRA_EINVAL, "negative cost parameters");
  if (c.kv_chunk_align < 0 || c.kv_chunk_min < 0) return fail(BSRA_EINVAL, "negative chunk parameters");
  if (c.kernel < BSRA_KERNEL_AUTO || c.kernel > BSRA_KERNEL_TC) return fail(BSRA_EINVAL, "bad kernel selector");
  if (c.flags & ~(BSRA_FLAG_PDL | BSRA_FLAG_RAGGED_KV | BSRA_FLAG_BALANCE_CTAS | BSRA_FLAG_CP_GATHER |
                  BSRA_FLAG_CP_ASYNC | BSRA_FLAG_DEFER_CONTRACTION))
    return fail(BSRA_EINVAL, "unknown flag bits");
  if ((c.flags & BSRA_FLAG_DEFER_CONTRACTION) && (tm & 14) == 0)
    return fail(BSRA_EINVAL, "BSRA_FLAG_DEFER_CONTRACTION: decode-only engines merge in-kernel (no contraction stage)");
  if ((c.flags & BSRA_FLAG_RAGGED_KV) && c.page_size != 128)
    return fail(BSRA_EINVAL, "BSRA_FLAG_RAGGED_KV engines take page_size = 128 (the KV tile)");
  if (c.sliding_window < 0) return fail(BSRA_EINVAL, "sliding_window < 0");
  if (!(c.logits_soft_cap >= 0.f) || !std::isfinite(c.logits_soft_cap))
    return fail(BSRA_EINVAL, "logits_soft_cap must be finite and >= 0");
  if (c.kv_dtype != 0 && c.kv_dtype != c.dtype && c.kv_dtype != BSRA_E4M3) return fail(BSRA_EINVAL, "bad kv_dtype");
  if (kv_is_f8(c) && c.dtype != BSRA_F16 && c.dtype != BSRA_BF16)
    return fail(BSRA_EINVAL, "an E4M3 KV cache takes F16 or BF16 q / o (P:499)");
  if (!(c.k_scale >= 0.f) || !std::isfinite(c.k_scale) || !(c.v_scale >= 0.f) || !std::isfinite(c.v_scale))
    return fail(BSRA_EINVAL, "k_scale / v_scale must be finite and >= 0");
  if (c.alibi != 0 && c.alibi != 1) return fail(BSRA_EINVAL, "alibi must be 0 or 1");
  if (c.max_total_kv_tokens < 0 || c.max_qo_len < 0) return fail(BSRA_EINVAL, "negative bounds");
  if (!(c.rope_theta >= 0.f) || !std::isfinite(c.rope_theta) || !(c.rope_scale >= 0.f) || !std::isfinite(c.rope_scale))
    return fail(BSRA_EINVAL, "rope_theta / rope_scale must be finite and >= 0");
  if (c.rope_theta > 0.f && kv_is_f8(c)) return fail(BSRA_EUNSUPPORTED, "RoPE with an E4M3 KV cache");
  for (int i = 0; i < 2; ++i)
    if (c.reserved[i]) return fail(BSRA_EINVAL, "reserved fields must be zero");
  return BSRA_OK;
}

int32_t default_num_ctas(const bsra_config& c, int32_t sms) {
  // one persistent CTA per SM (App. D.3: k = 1 "persistent kernel"); the SIMT decode
  // path fits two per SM, the tcgen05 kernels one.
  const bool decode = c.tile_q == 16 || (c.tile_q == 0 && tile_mask_of(c) == 1);
  const bool simt = c.kernel == BSRA_KERNEL_SIMT || c.dtype == BSRA_F32 || (kv_is_f8(c) && c.head_dim != 128);
  return decode && simt ? 2 * sms : sms;
}

Layout make_layout(const bsra_config& c, int32_t num_ctas) {
  Layout L;
  L.num_ctas = num_ctas;
  const int tm = c.tile_q ? (c.tile_q == 16 ? 1 : c.tile_q == 64 ? 2 : c.tile_q == 128 ? 4 : 8) : tile_mask_of(c);
  L.T_min = (tm & 1) ? 16 : (tm & 2) ? 64 : (tm & 4) ? 128 : 256;
  L.T_max = (tm & 8) ? 256 : (tm & 4) ? 128 : (tm & 2) ? 64 : 16;
  const int32_t g = c.num_qo_heads / c.num_kv_heads;
  L.plan_words = bsra::plan_capacity_words(num_ctas, c.num_kv_heads, g, c.max_batch, c.max_total_qo_rows, L.T_min);
  size_t off = 0;
  L.off_plan = off;
  off = align_up(off + L.plan_words * 4, 256);
  const size_t slots = 2 * (size_t)num_ctas;
  L.off_part_o = off;
  off = align_up(off + slots * L.T_max * c.head_dim * 4, 256);
  L.off_part_lse = off;
  off = align_up(off + slots * L.T_max * 4, 256);
  L.off_counters = off;
  off = align_up(off + (size_t)(num_ctas + 1) * 4, 256);
  L.off_aux = off;
  L.aux_words = 2 * ((size_t)c.max_batch + 1);
  off = align_up(off + L.aux_words * 4, 256);
  // fp8 KV with prefill tiles on the tcgen05 path: the 16-bit gather region (f8_gather.cuh),
  // caller-owned like the rest of the workspace (§8(b) ownership; never cudaMalloc'd by plan)
  L.off_f8 = off;
  if (kv_is_f8(c) && L.T_max > 16 && c.head_dim == 128 && c.kernel != BSRA_KERNEL_SIMT)
    L.f8_rows = c.max_total_kv_tokens;
  off = align_up(off + (size_t)L.f8_rows * c.num_kv_heads * 128 * 2 * sizeof(uint16_t), 256);
  // device planner: per request 3, per row 5, per item 2 words (rows <= items <= plan_words / 6)
  L.off_devscratch = off;
  L.devscratch_words = 2 * L.plan_words + 3 * ((size_t)c.max_batch + 1) + (size_t)num_ctas + 64;
  off = align_up(off + L.devscratch_words * 4, 256);
  L.total = off;
  return L;
}

bsra_status query_sms(int32_t device, int32_t* sms) {
  CUDA_TRY(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device));
  return BSRA_OK;
}

}  // namespace

// Launch choices a captured CUDA graph bakes in (bsra.h, bsra_run: graph capture)
struct LaunchSig {
  int32_t T_q = 0;
  int32_t kc = 0;           // decode kernel's live fused columns (4 / 8 / 16)
  bool f8_prefill = false;  // fp8 gather pass + 16-bit prefill kernel
  int64_t q_extent = 0;     // rows of the q tensor map
  int64_t kv_extent = 0;    // contiguous-KV token extent of the K/V maps
};

struct bsra_engine {
  bsra_config cfg;
  int32_t device = 0;
  int32_t sms = 148;  // SM count of `device` (grid sizes of the helper kernels)
  Layout lay;
  uint8_t* ws = nullptr;
  int32_t* staging = nullptr;  // pinned host buffer (App. D)
  cudaEvent_t staged = nullptr;  // guards staging reuse
  bool have_event_pending = false;
  std::vector<int32_t> image;  // host copy of the current plan
  bsra::PlanSummary summary;
  bool planned = false;
  bool counters_zeroed = false;
  float sm_scale = 0.f;
  int64_t total_qo = 0;
  int64_t total_kv = 0;  // ragged KV: token extent of k / v (kv_indptr[batch])
  int32_t max_qo = 0;
  int32_t kc = 16;  // decode kernel's live fused columns for the current plan
  float k_scale = 1.f, v_scale = 1.f;  // fp8 KV dequantisation scales (bsra_set_kv_scales)
  uint64_t rope_f[64] = {};            // RoPE: theta_i / 2pi in 2^-64 turns (R31), i < D/2
  // fp8 KV with prefill tiles (f8_gather.cuh): the current plan addresses a 16-bit gathered copy
  // in the workspace's f8 region ([2][lay.f8_rows, H_kv, 128])
  bool f8_prefill = false;
  int64_t f8_rows = 0;       // sum of l_kv of the current plan
  bool device_planned = false;  // the current plan was built on the device (bsra_plan_device)
  bool captured = false;     // a run() was captured into a CUDA graph since the last release
  LaunchSig cap_sig;         // launch choices of that captured run()
  long long* trace = nullptr;  // BSRA_EXPERIMENTS builds: device buffer for kernel pipeline traces
  bsra::AttnParams deferred{};  // BSRA_FLAG_DEFER_CONTRACTION: the last run's parameters (bsra_contract)
  bool have_deferred = false;
  int32_t last_launches = 0;
  const char* selected = "none";
};

// Definitions below take C linkage from their declarations in bsra.h.

int32_t bsra_version(void) { return 100; }

const char* bsra_last_error(void) { return g_err.c_str(); }

bsra_status bsra_num_sms(int32_t device, int32_t* out) {
  if (!out) return fail(BSRA_EINVAL, "NULL out");
  return query_sms(device, out);
}

bsra_status bsra_workspace_bytes(const bsra_config* cfg, int32_t device, size_t* device_bytes) {
  if (!cfg || !device_bytes) return fail(BSRA_EINVAL, "NULL argument");
  bsra_status s = validate_config(*cfg);
  if (s) return s;
  int32_t nc = cfg->num_ctas;
  if (!nc) {
    int32_t sms = 0;
    s = query_sms(device, &sms);
    if (s) return s;
    nc = default_num_ctas(*cfg, sms);
  }
  *device_bytes = make_layout(*cfg, nc).total;
  return BSRA_OK;
}

bsra_status bsra_engine_create(const bsra_config* cfg, int32_t device, void* d_workspace, size_t ws_bytes,
                               bsra_engine** out) {
  if (!cfg || !out) return fail(BSRA_EINVAL, "NULL argument");
  *out = nullptr;
  bsra_status s = validate_config(*cfg);
  if (s) return s;
  if (!d_workspace) return fail(BSRA_EINVAL, "NULL workspace");
  if (reinterpret_cast<uintptr_t>(d_workspace) % 256) return fail(BSRA_EINVAL, "workspace must be 256-byte aligned");
  int32_t nc = cfg->num_ctas;
  if (!nc) {
    int32_t sms = 0;
    s = query_sms(device, &sms);
    if (s) return s;
    nc = default_num_ctas(*cfg, sms);
  }
  Layout lay = make_layout(*cfg, nc);
  if (ws_bytes < lay.total)
    return fail(BSRA_ENOMEM, "workspace too small: need " + std::to_string(lay.total) + " bytes");
  auto* e = new (std::nothrow) bsra_engine();
  if (!e) return fail(BSRA_ENOMEM, "host allocation failed");
  e->cfg = *cfg;
  e->cfg.num_ctas = nc;
  e->k_scale = cfg->k_scale > 0.f ? cfg->k_scale : 1.f;
  e->v_scale = cfg->v_scale > 0.f ? cfg->v_scale : 1.f;
  if (cfg->rope_theta > 0.f) {  // RoPE frequencies as exact fractions of a turn: pos * F mod 2^64
    const long double two_pi = 6.283185307179586476925286766559L;
    const long double scale = cfg->rope_scale > 0.f ? (long double)cfg->rope_scale : 1.0L;
    for (int i = 0; i < cfg->head_dim / 2; ++i) {
      const long double theta = powl((long double)cfg->rope_theta, -2.0L * i / cfg->head_dim) / scale;
      e->rope_f[i] = (uint64_t)llroundl(ldexpl(theta / two_pi, 64));
    }
  }
  e->device = device;
  if (query_sms(device, &e->sms) != BSRA_OK) e->sms = 148;
  e->lay = lay;
  e->ws = static_cast<uint8_t*>(d_workspace);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  cudaError_t ce = cudaMallocHost(&e->staging, (lay.plan_words + lay.aux_words) * 4);
  if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&e->staged, cudaEventDisableTiming);
  cudaSetDevice(prev);
  if (ce != cudaSuccess) {
    if (e->staging) cudaFreeHost(e->staging);
    delete e;
    return fail(BSRA_ECUDA, std::string("pinned staging: ") + cudaGetErrorString(ce));
  }
  *out = e;
  return BSRA_OK;
}

void bsra_engine_destroy(bsra_engine* e) {
  if (!e) return;
  if (e->staged) {
    cudaEventSynchronize(e->staged);
    cudaEventDestroy(e->staged);
  }
  if (e->staging) cudaFreeHost(e->staging);
  delete e;
}

static bsra::SchedParams sched_params(const bsra_config& c, int32_t num_ctas) {
  bsra::SchedParams sp;
  sp.H_qo = c.num_qo_heads;
  sp.H_kv = c.num_kv_heads;
  sp.page_size = c.page_size;
  sp.mask = c.mask;
  sp.num_ctas = num_ctas;
  sp.tile_set_mask = tile_mask_of(c);
  sp.tile_q = c.tile_q;
  sp.alpha = c.cost_alpha ? c.cost_alpha : 1;
  sp.beta = c.cost_beta ? c.cost_beta : 1;
  sp.align = c.kv_chunk_align ? c.kv_chunk_align : c.page_size;
  sp.L_min = c.kv_chunk_min;
  sp.window = c.sliding_window;
  return sp;
}

bsra_status bsra_plan_host(const bsra_config* cfg, int32_t num_ctas, int32_t batch, const int32_t* qo_indptr,
                           const int32_t* kv_page_indptr, const int32_t* kv_last_page_len, int32_t* image,
                           size_t cap_words, size_t* n_words) {
  if (!cfg || !n_words) return fail(BSRA_EINVAL, "NULL argument");
  bsra_status s = validate_config(*cfg);
  if (s) return s;
  if (num_ctas < 1) return fail(BSRA_EINVAL, "num_ctas < 1");
  std::vector<int32_t> qo, kv, im;
  std::string err = bsra::lengths_from_bsr(batch, qo_indptr, kv_page_indptr, kv_last_page_len, cfg->page_size, qo, kv);
  if (!err.empty()) return fail(BSRA_EINVAL, err);
  bsra::PlanSummary sum;
  err = bsra::build_plan(sched_params(*cfg, num_ctas), qo, kv, qo_indptr, kv_page_indptr, im, sum);
  if (!err.empty()) return fail(BSRA_EINVAL, err);
  *n_words = im.size();
  if (image) {
    if (cap_words < im.size()) return fail(BSRA_ENOMEM, "image buffer too small");
    std::memcpy(image, im.data(), im.size() * 4);
  }
  return BSRA_OK;
}

namespace {

// Shared inspector core: Algorithm 1 over (qo, kv) lengths; `page_begin` gives each request's
// first BSR page (paged) or first token row (contiguous KV) for the plan's request table.
// fp8 KV with a prefill tile (T_q > 16) on the tcgen05 path: the plan is re-encoded with each
// request's first row in the gathered 16-bit copy (f8_gather.cuh) and `page_begin` goes to the
// aux section for the gather pass.
// Makespan of a plan image under the Algorithm-1 cost model (alpha*T_q + beta*chunk per item).
int64_t image_makespan(const std::vector<int32_t>& im, int64_t alpha, int64_t beta) {
  const int nc = im[2], T_q = im[3], n_items = im[5];
  const int32_t* ind = im.data() + bsra::kHeaderWords;
  const int32_t* kb = ind + nc + 1 + 3 * n_items;
  const int32_t* ke = kb + n_items;
  int64_t mx = 0;
  for (int c = 0; c < nc; ++c) {
    int64_t s = 0;
    for (int it = ind[c]; it < ind[c + 1]; ++it) s += alpha * T_q + beta * (int64_t)(ke[it] - kb[it]);
    mx = std::max(mx, s);
  }
  return mx;
}

// Re-encodes an image planned with c queues for a grid of nc >= c CTAs: queues c..nc-1 empty.
void pad_queues(std::vector<int32_t>& im, int32_t nc) {
  const int32_t c = im[2];
  if (c == nc) return;
  const int32_t n_items = im[bsra::kHeaderWords + c];  // cta_indptr[c]
  im[2] = nc;
  im.insert(im.begin() + bsra::kHeaderWords + c + 1, (size_t)(nc - c), n_items);
}

bool is_ragged_engine(const bsra_engine* e) { return (e->cfg.flags & BSRA_FLAG_RAGGED_KV) != 0; }
int64_t ragged_total(const std::vector<int32_t>& kv) {
  int64_t t = 0;
  for (int32_t x : kv) t += x;
  return t;
}

bsra_status plan_core(bsra_engine* e, const int32_t* qo_indptr, const int32_t* page_begin,
                      const std::vector<int32_t>& qo, const std::vector<int32_t>& kv, float sm_scale, void* stream) {
  const bsra_config& c = e->cfg;
  int64_t rows = 0;
  for (int32_t x : qo) rows += x;
  if (rows > c.max_total_qo_rows) return fail(BSRA_EBOUNDS, "sum of qo lengths exceeds max_total_qo_rows");
  std::vector<int32_t> im;
  bsra::PlanSummary sum;
  int32_t queues = c.num_ctas;  // Algorithm 1's #CTA (BSRA_FLAG_BALANCE_CTAS may pick fewer)
  std::string err = bsra::build_plan(sched_params(c, queues), qo, kv, qo_indptr, page_begin, im, sum);
  if (!err.empty()) return fail(BSRA_EINVAL, err);
  if (c.flags & BSRA_FLAG_BALANCE_CTAS) {
    const int64_t alpha = c.cost_alpha ? c.cost_alpha : 1, beta = c.cost_beta ? c.cost_beta : 1;
    int64_t best = image_makespan(im, alpha, beta);
    for (int32_t q = c.num_ctas - 1; q >= std::max(1, c.num_ctas - c.num_ctas / 8); --q) {
      std::vector<int32_t> im2;
      bsra::PlanSummary s2;
      err = bsra::build_plan(sched_params(c, q), qo, kv, qo_indptr, page_begin, im2, s2);
      if (!err.empty()) return fail(BSRA_EINVAL, err);
      const int64_t mk = image_makespan(im2, alpha, beta);
      if (mk < best) {
        best = mk;
        queues = q;
        im.swap(im2);
        sum = s2;
      }
    }
  }
  const int32_t batch = (int32_t)qo.size();
  const int32_t g = c.num_qo_heads / c.num_kv_heads;
  const bool f8_prefill = kv_is_f8(c) && sum.T_q > 16 && c.kernel != BSRA_KERNEL_SIMT && c.head_dim == 128 &&
                          (g & (g - 1)) == 0;
  int32_t max_qo = 0;
  for (int32_t x : qo) max_qo = std::max(max_qo, x);
  if (c.max_qo_len > 0 && max_qo > c.max_qo_len) return fail(BSRA_EBOUNDS, "a request's l_qo exceeds max_qo_len");
  const int64_t fused = std::min<int64_t>(16, (int64_t)(c.max_qo_len > 0 ? c.max_qo_len : max_qo) * g);
  const int32_t kc = fused <= 4 ? 4 : fused <= 8 ? 8 : 16;
  std::vector<int32_t> kv_off;
  int64_t f8_rows = 0;
  if (f8_prefill) {
    kv_off.resize(batch + 1, 0);
    for (int32_t i = 0; i < batch; ++i) {
      f8_rows += kv[i];
      if (f8_rows > INT32_MAX) return fail(BSRA_EBOUNDS, "fp8 prefill: more than 2^31 KV tokens in one plan");
      kv_off[i + 1] = (int32_t)f8_rows;
    }
    err = bsra::build_plan(sched_params(c, queues), qo, kv, qo_indptr, kv_off.data(), im, sum);
    if (!err.empty()) return fail(BSRA_EINVAL, err);
  }
  pad_queues(im, c.num_ctas);
  if (im.size() > e->lay.plan_words) return fail(BSRA_EBOUNDS, "plan image exceeds the workspace plan section");
  if (sum.T_q > e->lay.T_max) return fail(BSRA_EBOUNDS, "tile larger than the workspace partial slots");
  if (f8_prefill && f8_rows > e->lay.f8_rows)
    return fail(BSRA_EBOUNDS, "fp8 KV with prefill tiles: sum of l_kv (" + std::to_string(f8_rows) +
                                  ") exceeds max_total_kv_tokens (" + std::to_string(e->lay.f8_rows) +
                                  "), the workspace's 16-bit gather region");
  if (e->captured) {  // a CUDA graph holds the launch choices of an earlier plan (bsra.h, bsra_run)
    const LaunchSig& k = e->cap_sig;
    std::string why;
    if (sum.T_q != k.T_q) why = "query tile T_q " + std::to_string(k.T_q) + " -> " + std::to_string(sum.T_q);
    else if (sum.T_q == 16 && kc > k.kc) why = "decode live columns " + std::to_string(k.kc) + " -> " + std::to_string(kc);
    else if (f8_prefill != k.f8_prefill) why = "fp8 gather pass";
    else if (rows > k.q_extent) why = "q rows beyond the captured tensor-map extent";
    else if (is_ragged_engine(e) && ragged_total(kv) > k.kv_extent) why = "KV tokens beyond the captured extent";
    if (!why.empty())
      return fail(BSRA_EBOUNDS, "re-plan changes a launch choice baked into a captured CUDA graph (" + why +
                                    "); destroy the graph, call bsra_graph_release and re-capture");
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the previous upload must have left the pinned buffer before it is overwritten
  if (e->have_event_pending) CUDA_TRY(cudaEventSynchronize(e->staged));
  std::memcpy(e->staging, im.data(), im.size() * 4);
  CUDA_TRY(cudaMemcpyAsync(e->ws + e->lay.off_plan, e->staging, im.size() * 4, cudaMemcpyHostToDevice, st));
  if (f8_prefill) {  // aux: src_begin[batch+1] at 0, kv_off[batch+1] at max_batch+1
    int32_t* aux = e->staging + e->lay.plan_words;
    const size_t stride = (size_t)c.max_batch + 1;
    std::memcpy(aux, page_begin, (size_t)(batch + 1) * 4);
    std::memcpy(aux + stride, kv_off.data(), (size_t)(batch + 1) * 4);
    CUDA_TRY(cudaMemcpyAsync(e->ws + e->lay.off_aux, aux, e->lay.aux_words * 4, cudaMemcpyHostToDevice, st));
  }
  CUDA_TRY(cudaEventRecord(e->staged, st));
  e->have_event_pending = true;
  if (!e->counters_zeroed) {  // merge-list arrival counters start at 0; the merging CTA resets them
    CUDA_TRY(cudaMemsetAsync(e->ws + e->lay.off_counters, 0, (size_t)(e->lay.num_ctas + 1) * 4, st));
    e->counters_zeroed = true;
  }
  e->image.swap(im);
  e->summary = sum;
  e->planned = true;
  e->have_deferred = false;  // bsra_contract needs a run of this plan
  e->device_planned = false;
  e->f8_prefill = f8_prefill;
  e->f8_rows = f8_rows;
  e->sm_scale = sm_scale > 0.f ? sm_scale : 1.f / std::sqrt((float)c.head_dim);
  e->total_qo = rows;
  e->max_qo = max_qo;
  e->kc = kc;
  return BSRA_OK;
}

}  // namespace

bsra_status bsra_plan(bsra_engine* e, int32_t batch, const int32_t* qo_indptr, const int32_t* kv_page_indptr,
                      const int32_t* kv_last_page_len, float sm_scale, void* stream) {
  if (!e) return fail(BSRA_EINVAL, "NULL engine");
  const bsra_config& c = e->cfg;
  if (c.flags & BSRA_FLAG_RAGGED_KV) return fail(BSRA_EINVAL, "contiguous-KV engine: use bsra_plan_ragged");
  if (batch > c.max_batch) return fail(BSRA_EBOUNDS, "batch exceeds max_batch");
  std::vector<int32_t> qo, kv;
  std::string err = bsra::lengths_from_bsr(batch, qo_indptr, kv_page_indptr, kv_last_page_len, c.page_size, qo, kv);
  if (!err.empty()) return fail(BSRA_EINVAL, err);
  return plan_core(e, qo_indptr, kv_page_indptr, qo, kv, sm_scale, stream);
}

bsra_status bsra_plan_device(bsra_engine* e, int32_t batch, const int32_t* d_qo_indptr, const int32_t* d_kv_page_indptr,
                             const int32_t* d_kv_last_page_len, float sm_scale, void* stream) {
  if (!e) return fail(BSRA_EINVAL, "NULL engine");
  const bsra_config& c = e->cfg;
  if (c.flags & BSRA_FLAG_RAGGED_KV) return fail(BSRA_EUNSUPPORTED, "device planning: paged engines only");
  if (c.flags & BSRA_FLAG_BALANCE_CTAS) return fail(BSRA_EUNSUPPORTED, "device planning: no BSRA_FLAG_BALANCE_CTAS");
  if (!c.tile_q) return fail(BSRA_EUNSUPPORTED, "device planning needs a fixed tile (cfg.tile_q)");
  if (c.tile_q == 16 && c.max_qo_len <= 0)
    return fail(BSRA_EUNSUPPORTED, "device planning of decode tiles needs cfg.max_qo_len");
  if (kv_is_f8(c) && c.tile_q > 16) return fail(BSRA_EUNSUPPORTED, "device planning: no fp8 prefill tiles");
  if (c.num_ctas > 512) return fail(BSRA_EUNSUPPORTED, "device planning: num_ctas > 512");
  const int64_t alpha = c.cost_alpha ? c.cost_alpha : 1, beta = c.cost_beta ? c.cost_beta : 1;
  if (alpha > (1 << 20) || beta > (1 << 20)) return fail(BSRA_EUNSUPPORTED, "device planning: alpha / beta > 2^20");
  if (batch < 0) return fail(BSRA_EINVAL, "batch < 0");
  if (batch > c.max_batch) return fail(BSRA_EBOUNDS, "batch exceeds max_batch");
  if (batch > 0 && (!d_qo_indptr || !d_kv_page_indptr || !d_kv_last_page_len)) return fail(BSRA_EINVAL, "NULL array");
  if (e->captured && e->cap_sig.T_q != c.tile_q)
    return fail(BSRA_EBOUNDS, "re-plan changes a launch choice baked into a captured CUDA graph (query tile)");
  bsra::DevPlanParams P{};
  P.qo_indptr = d_qo_indptr;
  P.kv_page_indptr = d_kv_page_indptr;
  P.kv_last_page_len = d_kv_last_page_len;
  P.image = reinterpret_cast<int32_t*>(e->ws + e->lay.off_plan);
  P.scratch = reinterpret_cast<int32_t*>(e->ws + e->lay.off_devscratch);
  P.scratch_words = (int64_t)e->lay.devscratch_words;
  P.cap_words = (int32_t)e->lay.plan_words;
  P.batch = batch;
  P.H_kv = c.num_kv_heads;
  P.g = c.num_qo_heads / c.num_kv_heads;
  P.page_size = c.page_size;
  P.mask = c.mask;
  P.num_ctas = c.num_ctas;
  P.T_q = c.tile_q;
  P.align = c.kv_chunk_align ? c.kv_chunk_align : c.page_size;
  P.L_min = c.kv_chunk_min;
  P.window = c.sliding_window;
  P.max_total_qo_rows = c.max_total_qo_rows;
  P.alpha = alpha;
  P.beta = beta;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(bsra::plan_device_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  bsra::devplan::kSmemBytes));
    attr = true;
  }
  bsra::plan_device_kernel<<<1, bsra::devplan::kThreads, bsra::devplan::kSmemBytes, st>>>(P);
  CUDA_TRY(cudaGetLastError());
  if (!e->counters_zeroed) {
    CUDA_TRY(cudaMemsetAsync(e->ws + e->lay.off_counters, 0, (size_t)(e->lay.num_ctas + 1) * 4, st));
    e->counters_zeroed = true;
  }
  // host-side launch choices from the engine bounds (the plan itself stays on the device)
  const int32_t g = c.num_qo_heads / c.num_kv_heads;
  const int64_t fused = std::min<int64_t>(16, (int64_t)std::max(1, c.max_qo_len) * g);
  e->image.clear();
  e->summary = bsra::PlanSummary();
  e->summary.T_q = c.tile_q;
  e->summary.n_items = 1;  // unknown on the host: run() validates its pointers
  e->planned = true;
  e->have_deferred = false;  // bsra_contract needs a run of this plan
  e->device_planned = true;
  e->f8_prefill = false;
  e->f8_rows = 0;
  e->sm_scale = sm_scale > 0.f ? sm_scale : 1.f / std::sqrt((float)c.head_dim);
  e->total_qo = c.max_total_qo_rows;
  e->max_qo = c.max_qo_len;
  e->kc = fused <= 4 ? 4 : fused <= 8 ? 8 : 16;
  return BSRA_OK;
}

bsra_status bsra_plan_device_status(bsra_engine* e, void* stream, int32_t* code) {
  if (!e || !code) return fail(BSRA_EINVAL, "NULL argument");
  if (!e->device_planned) {
    *code = 0;
    return BSRA_OK;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t hdr[16];
  CUDA_TRY(cudaMemcpyAsync(hdr, e->ws + e->lay.off_plan, sizeof(hdr), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *code = hdr[12];
  return BSRA_OK;
}

bsra_status bsra_plan_ragged(bsra_engine* e, int32_t batch, const int32_t* qo_indptr, const int32_t* kv_indptr,
                             float sm_scale, void* stream) {
  if (!e) return fail(BSRA_EINVAL, "NULL engine");
  const bsra_config& c = e->cfg;
  if (!(c.flags & BSRA_FLAG_RAGGED_KV)) return fail(BSRA_EINVAL, "paged engine: use bsra_plan (or create with BSRA_FLAG_RAGGED_KV)");
  if (batch < 0) return fail(BSRA_EINVAL, "batch < 0");
  if (batch > c.max_batch) return fail(BSRA_EBOUNDS, "batch exceeds max_batch");
  if (batch > 0 && (!qo_indptr || !kv_indptr)) return fail(BSRA_EINVAL, "NULL indptr");
  std::vector<int32_t> qo(batch), kv(batch);
  if (batch > 0 && (qo_indptr[0] != 0 || kv_indptr[0] != 0)) return fail(BSRA_EINVAL, "indptr[0] != 0");
  for (int32_t i = 0; i < batch; ++i) {
    qo[i] = qo_indptr[i + 1] - qo_indptr[i];
    kv[i] = kv_indptr[i + 1] - kv_indptr[i];
    if (qo[i] < 0) return fail(BSRA_EINVAL, "qo_indptr not nondecreasing at " + std::to_string(i));
    if (kv[i] < 0) return fail(BSRA_EINVAL, "kv_indptr not nondecreasing at " + std::to_string(i));
  }
  bsra_status s = plan_core(e, qo_indptr, kv_indptr, qo, kv, sm_scale, stream);
  if (s) return s;
  e->total_kv = batch > 0 ? kv_indptr[batch] : 0;
  return BSRA_OK;
}

namespace {

template <typename T, typename TKV, int D>
bsra_status launch_simt(const bsra::AttnParams& p, int grid, cudaStream_t st) {
  using S = bsra::SimtSmem<TKV, D>;
  static bool attr = false;
  if (!attr) {
    CUDA_TRY(cudaFuncSetAttribute(bsra::attn_simt_kernel<T, TKV, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  S::kBytes));
    attr = true;
  }
  bsra::attn_simt_kernel<T, TKV, D><<<grid, bsra::kSimtWarps * 32, S::kBytes, st>>>(p);
  CUDA_TRY(cudaGetLastError());
  return BSRA_OK;
}

template <typename T, typename TKV = T>
bsra_status launch_simt_d(const bsra::AttnParams& p, int D, int grid, cudaStream_t st) {
  return D == 64 ? launch_simt<T, TKV, 64>(p, grid, st) : launch_simt<T, TKV, 128>(p, grid, st);
}

template <typename TO, int D>
bsra_status launch_contraction_t(const bsra::AttnParams& p, int grid, cudaStream_t st, bool pdl) {
  // pdl: programmatic dependent launch — the kernel's blocks start (plan and list reads) while
  // the attention kernel before it drains, and wait (griddepcontrol.wait) before the partials
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? attr : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, bsra::contraction_kernel<TO, D>, p));
  return BSRA_OK;
}

// Contraction grid: one warp per (list, row) up to a full GPU of 256-thread blocks (the stage is
// latency-bound: each warp's slot loads are one dependent round trip). Fixed per engine (lists <=
// num_ctas, rows <= T_max), so captured graphs stay valid across re-plans.
int contraction_grid(const bsra_engine* e) {
  const int64_t warps = (int64_t)e->cfg.num_ctas * e->lay.T_max;
  return (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, 8 * (int64_t)e->sms));
}

template <typename TO>
bsra_status launch_contraction_d(const bsra::AttnParams& p, int D, int grid, cudaStream_t st, bool pdl) {
  return D == 64 ? launch_contraction_t<TO, 64>(p, grid, st, pdl) : launch_contraction_t<TO, 128>(p, grid, st, pdl);
}

}  // namespace

namespace {

// Shared executor core. Paged: k_strides = (page, slot, head) and the BSR page ids. Contiguous KV
// (ragged): k_strides = (token, token, head), no page ids; token t of request i is row
// kv_indptr[i] + t (the plan's page_begin).
bsra_status run_core(bsra_engine* e, const void* q, const void* k_pool, const void* v_pool, const int64_t* k_strides,
                     const int64_t* v_strides, const int32_t* kv_page_indices, bool ragged, const uint8_t* custom_mask,
                     const int64_t* mask_bit_indptr, void* o, float* lse, void* stream) {
  if (!e->planned) return fail(BSRA_EINVAL, "run() before plan()");
  const bsra_config& c = e->cfg;
  e->last_launches = 0;
  const bool has_rows = e->summary.n_items > 0;
  if (has_rows && (!q || !k_pool || !v_pool || (!ragged && !kv_page_indices) || !o))
    return fail(BSRA_EINVAL, "NULL tensor pointer");
  if (c.mask == BSRA_MASK_CUSTOM && has_rows && (!custom_mask || !mask_bit_indptr))
    return fail(BSRA_EINVAL, "MASK_CUSTOM needs custom_mask and mask_bit_indptr");
  const int es = dtype_size(kv_dtype_of(c));
  for (int i = 0; i < 3; ++i)
    if ((k_strides[i] * es) % 16 || (v_strides[i] * es) % 16 || k_strides[i] < 0 || v_strides[i] < 0)
      return fail(BSRA_EINVAL, "pool strides must be non-negative and 16-byte multiples");
  if (has_rows && ((reinterpret_cast<uintptr_t>(k_pool) | reinterpret_cast<uintptr_t>(v_pool) |
                    reinterpret_cast<uintptr_t>(q)) % 16))
    return fail(BSRA_EINVAL, "q and the pools must be 16-byte aligned");
  if (has_rows && reinterpret_cast<uintptr_t>(o) % 32)
    return fail(BSRA_EINVAL, "o must be 32-byte aligned (256-bit row stores)");

  bsra::AttnParams p{};
  p.plan = reinterpret_cast<const int32_t*>(e->ws + e->lay.off_plan);
  p.q = q;
  p.k = k_pool;
  p.v = v_pool;
  p.ks0 = k_strides[0];
  p.ks1 = k_strides[1];
  p.ks2 = k_strides[2];
  p.vs0 = v_strides[0];
  p.vs1 = v_strides[1];
  p.vs2 = v_strides[2];
  p.page_indices = kv_page_indices;
  p.kv_ragged = ragged ? 1 : 0;
  p.window = c.sliding_window;
  // fp8 KV (R28): k = k_scale * E4M3(byte) folds into the logit scale; v_scale scales o
  const float logit_scale = e->sm_scale * (kv_is_f8(c) ? e->k_scale : 1.f);
  p.kv_f8 = kv_is_f8(c) ? 1 : 0;
  p.v_scale = kv_is_f8(c) ? e->v_scale : 1.f;
  // soft-cap in raw q.k units: c * tanh(sm_scale*s / c) = sm_scale * c' tanh(s / c'), c' = c / sm_scale
  p.soft_cap = c.logits_soft_cap > 0.f ? c.logits_soft_cap / logit_scale : 0.f;
  p.inv_soft_cap = c.logits_soft_cap > 0.f ? logit_scale / c.logits_soft_cap : 0.f;
  p.mask = custom_mask;
  p.mask_indptr = mask_bit_indptr;
  p.o = o;
  p.lse = lse;
  p.part_o = reinterpret_cast<float*>(e->ws + e->lay.off_part_o);
  p.part_lse = reinterpret_cast<float*>(e->ws + e->lay.off_part_lse);
  p.counters = reinterpret_cast<int32_t*>(e->ws + e->lay.off_counters);
  p.trace = e->trace;
  // Contraction placement, fixed per engine so a captured graph is valid for every re-plan:
  // decode engines (tiles of <= 16 rows) merge split items in-kernel (the CTA completing a list
  // folds it); engines that can emit 64/128-row tiles use the wide contraction kernel.
  p.fused_merge = e->lay.T_max <= 16 ? 1 : 0;
  p.H_qo = c.num_qo_heads;
  p.H_kv = c.num_kv_heads;
  p.g = c.num_qo_heads / c.num_kv_heads;
  p.page_size = c.page_size;
  p.mask_mode = c.mask;
  p.o_f32 = c.o_dtype == BSRA_F32;
  p.T_slot = e->lay.T_max;
  p.D = c.head_dim;
  p.scale_log2 = logit_scale * bsra::kLog2e;
  p.alibi = c.alibi;
  p.inv_logit_scale = 1.f / logit_scale;  // ALiBi bias in raw q.k units (R30)
  p.rope = c.rope_theta > 0.f ? 1 : 0;
  std::memcpy(p.rope_f, e->rope_f, sizeof(p.rope_f));

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = c.num_ctas;
  bsra_status s = BSRA_OK;
  const int T_q = e->summary.T_q;
  cudaStreamCaptureStatus cap_status = cudaStreamCaptureStatusNone;
  CUDA_TRY(cudaStreamIsCapturing(st, &cap_status));
  const bool capturing = cap_status != cudaStreamCaptureStatusNone;
  // tensor-map extents: the plan's exact sizes, or under capture the engine bounds, so a replay
  // after a re-plan within the bounds still covers every row (bsra.h, bsra_run)
  const int64_t q_extent = capturing ? std::max<int64_t>(c.max_total_qo_rows, e->total_qo) : e->total_qo;
  int64_t kv_extent = e->total_kv;
  if (ragged && capturing && c.max_total_kv_tokens > 0) kv_extent = std::max<int64_t>(c.max_total_kv_tokens, kv_extent);
  if (e->f8_prefill) kv_extent = e->lay.f8_rows;  // the workspace gather region's rows
  bool used_tc = false;
  int gather_launches = 0;
  bool kv16 = !kv_is_f8(c);  // the attention kernel reads 16-bit (or f32) K/V
  if (e->f8_prefill) {
    // fp8 KV, prefill tiles: dequantise-and-gather the plan's tokens into the engine's 16-bit
    // copy, then run the 16-bit kernels on it as contiguous KV (f8_gather.cuh)
    bsra::F8GatherParams gp{};
    gp.k = static_cast<const uint8_t*>(k_pool);
    gp.v = static_cast<const uint8_t*>(v_pool);
    gp.ks0 = k_strides[0];
    gp.ks1 = k_strides[1];
    gp.ks2 = k_strides[2];
    gp.vs0 = v_strides[0];
    gp.vs1 = v_strides[1];
    gp.vs2 = v_strides[2];
    gp.page_indices = ragged ? nullptr : kv_page_indices;
    const int32_t* aux = reinterpret_cast<const int32_t*>(e->ws + e->lay.off_aux);
    gp.src_begin = aux;
    gp.kv_off = aux + c.max_batch + 1;
    gp.plan = p.plan;
    gp.page_size = c.page_size;
    gp.H_kv = c.num_kv_heads;
    gp.f16 = c.dtype == BSRA_F16;
    const int64_t plane = e->lay.f8_rows * c.num_kv_heads * 128;
    uint16_t* f8_buf = reinterpret_cast<uint16_t*>(e->ws + e->lay.off_f8);
    gp.ko = f8_buf;
    gp.vo = f8_buf + plane;
    bsra::f8_gather_kernel<<<4 * e->sms, 256, 0, st>>>(gp);
    CUDA_TRY(cudaGetLastError());
    gather_launches = 1;
    p.k = gp.ko;
    p.v = gp.vo;
    p.ks0 = p.ks1 = p.vs0 = p.vs1 = (int64_t)c.num_kv_heads * 128;
    p.ks2 = p.vs2 = 128;
    p.kv_ragged = 1;
    ragged = true;
    kv16 = true;
  }
  if (c.kernel != BSRA_KERNEL_SIMT && c.dtype != BSRA_F32) {
    bsra::TcLaunch tl;
    tl.f16 = c.dtype == BSRA_F16;
    tl.T_q = T_q;
    tl.grid = grid;
    tl.total_qo = q_extent;
    tl.align = c.kv_chunk_align ? c.kv_chunk_align : c.page_size;
    tl.page_size = c.page_size;
    tl.kc = e->kc;
    tl.mask = c.mask;
    // PDL lets the kernel start before its predecessor drains; the fp8 prefill kernel reads the
    // 16-bit copy the gather kernel right before it writes, so it is launched fully serialised
    tl.pdl = (c.flags & BSRA_FLAG_PDL) != 0 && !e->f8_prefill;
    tl.ragged = ragged;
    tl.total_kv = kv_extent;
    tl.f8kv = !kv16;
    tl.rope = p.rope != 0;
    tl.force_cp = (c.flags & (BSRA_FLAG_CP_GATHER | BSRA_FLAG_CP_ASYNC)) != 0;
    tl.force_cp_async = (c.flags & BSRA_FLAG_CP_ASYNC) != 0;
    const char* why = "";
    int rc = bsra::tc_launch(p, tl, st, &e->selected, &why);
    if (rc < 0)
      return fail(BSRA_ECUDA, std::string("tcgen05 kernel launch failed: ") + why + " / " +
                                  cudaGetErrorString(cudaGetLastError()));
    used_tc = rc > 0;
    if (!used_tc && c.kernel == BSRA_KERNEL_TC) return fail(BSRA_EUNSUPPORTED, std::string("no tcgen05 kernel: ") + why);
  }
  if (!used_tc) {
    e->selected = "simt";
    if (!kv16) {
      if (c.dtype == BSRA_F16) s = launch_simt_d<__half, __nv_fp8_e4m3>(p, c.head_dim, grid, st);
      else s = launch_simt_d<__nv_bfloat16, __nv_fp8_e4m3>(p, c.head_dim, grid, st);
    } else {
      switch (c.dtype) {
        case BSRA_F32: s = launch_simt_d<float>(p, c.head_dim, grid, st); break;
        case BSRA_F16: s = launch_simt_d<__half>(p, c.head_dim, grid, st); break;
        default: s = launch_simt_d<__nv_bfloat16>(p, c.head_dim, grid, st); break;
      }
    }
    if (s) return s;
  }
  e->last_launches = 1 + gather_launches;
  if (!p.fused_merge && (c.flags & BSRA_FLAG_DEFER_CONTRACTION)) {  // bsra_contract runs the stage
    e->deferred = p;
    e->have_deferred = true;
  } else if (!p.fused_merge) {  // contraction stage: fixed grid, exits at once if nothing split
    const int cgrid = contraction_grid(e);
    const bool pdl = (c.flags & BSRA_FLAG_PDL) != 0;
    if (c.o_dtype == BSRA_F32 || c.dtype == BSRA_F32) s = launch_contraction_d<float>(p, c.head_dim, cgrid, st, pdl);
    else if (c.dtype == BSRA_F16) s = launch_contraction_d<__half>(p, c.head_dim, cgrid, st, pdl);
    else s = launch_contraction_d<__nv_bfloat16>(p, c.head_dim, cgrid, st, pdl);
    if (s) return s;
    e->last_launches = 2 + gather_launches;
  }
  if (capturing) {  // record what the graph baked in; later plans are checked against it
    LaunchSig k;
    k.T_q = T_q;
    k.kc = e->kc;
    k.f8_prefill = e->f8_prefill;
    k.q_extent = q_extent;
    k.kv_extent = ragged && !e->f8_prefill ? kv_extent : INT64_MAX;
    if (e->captured) {  // several captures: keep the most restrictive choices
      k.kc = std::min(k.kc, e->cap_sig.kc);
      k.q_extent = std::min(k.q_extent, e->cap_sig.q_extent);
      k.kv_extent = std::min(k.kv_extent, e->cap_sig.kv_extent);
    }
    e->cap_sig = k;
    e->captured = true;
  }
  return BSRA_OK;
}

}  // namespace

bsra_status bsra_run(bsra_engine* e, const void* q, const void* k_pool, const void* v_pool, const int64_t* k_strides,
                     const int64_t* v_strides, const int32_t* kv_page_indices, const uint8_t* custom_mask,
                     const int64_t* mask_bit_indptr, void* o, float* lse, void* stream) {
  if (!e) return fail(BSRA_EINVAL, "NULL engine");
  if (e->cfg.flags & BSRA_FLAG_RAGGED_KV) return fail(BSRA_EINVAL, "contiguous-KV engine: use bsra_run_ragged");
  if (!k_strides || !v_strides) return fail(BSRA_EINVAL, "NULL strides");
  return run_core(e, q, k_pool, v_pool, k_strides, v_strides, kv_page_indices, false, custom_mask, mask_bit_indptr, o,
                  lse, stream);
}

bsra_status bsra_run_ragged(bsra_engine* e, const void* q, const void* k, const void* v, const int64_t* k_strides,
                            const int64_t* v_strides, const uint8_t* custom_mask, const int64_t* mask_bit_indptr,
                            void* o, float* lse, void* stream) {
  if (!e) return fail(BSRA_EINVAL, "NULL engine");
  if (!(e->cfg.flags & BSRA_FLAG_RAGGED_KV)) return fail(BSRA_EINVAL, "paged engine: use bsra_run");
  if (!k_strides || !v_strides) return fail(BSRA_EINVAL, "NULL strides");
  const int64_t ks[3] = {k_strides[0], k_strides[0], k_strides[1]};
  const int64_t vs[3] = {v_strides[0], v_strides[0], v_strides[1]};
  return run_core(e, q, k, v, ks, vs, nullptr, true, custom_mask, mask_bit_indptr, o, lse, stream);
}

bsra_status bsra_graph_release(bsra_engine* e) {
  if (!e) return fail(BSRA_EINVAL, "NULL engine");
  e->captured = false;
  e->cap_sig = LaunchSig();
  return BSRA_OK;
}

bsra_status bsra_set_kv_scales(bsra_engine* e, float k_scale, float v_scale) {
  if (!e) return fail(BSRA_EINVAL, "NULL engine");
  if (!(k_scale >= 0.f) || !std::isfinite(k_scale) || !(v_scale >= 0.f) || !std::isfinite(v_scale))
    return fail(BSRA_EINVAL, "k_scale / v_scale must be finite and >= 0");
  e->k_scale = k_scale > 0.f ? k_scale : 1.f;
  e->v_scale = v_scale > 0.f ? v_scale : 1.f;
  return BSRA_OK;
}

int32_t bsra_last_run_launches(const bsra_engine* e) { return e ? e->last_launches : 0; }

// Debug hook (not part of the public header): kernels that support tracing record CTA 0's
// pipeline events into this device buffer (NULL disables). See scripts/trace_prefill.py.
extern "C" void bsra_debug_set_trace(bsra_engine* e, long long* dev_buf) {
  if (e) e->trace = dev_buf;
}

const char* bsra_selected_kernel(const bsra_engine* e) { return e ? e->selected : "none"; }

namespace {
template <typename TI, typename TO, int D>
bsra_status merge_states_t(const void* oa, const float* la, const void* ob, const float* lb, int64_t n, void* out,
                           float* lo, cudaStream_t st) {
  if (n == 0) return BSRA_OK;
  const int grid = (int)std::min<int64_t>((n + 7) / 8, 148 * 16);  // grid-stride loop: any size works
  bsra::merge_states_kernel<TI, TO, D><<<grid, 256, 0, st>>>(static_cast<const TI*>(oa), la, static_cast<const TI*>(ob),
                                                              lb, n, static_cast<TO*>(out), lo);
  CUDA_TRY(cudaGetLastError());
  return BSRA_OK;
}
template <typename TI, typename TO>
bsra_status merge_states_d(int D, const void* oa, const float* la, const void* ob, const float* lb, int64_t n,
                           void* out, float* lo, cudaStream_t st) {
  return D == 64 ? merge_states_t<TI, TO, 64>(oa, la, ob, lb, n, out, lo, st)
                 : merge_states_t<TI, TO, 128>(oa, la, ob, lb, n, out, lo, st);
}
template <typename TI>
bsra_status merge_states_o(bsra_dtype to, int D, const void* oa, const float* la, const void* ob, const float* lb,
                           int64_t n, void* out, float* lo, cudaStream_t st) {
  switch (to) {
    case BSRA_F32: return merge_states_d<TI, float>(D, oa, la, ob, lb, n, out, lo, st);
    case BSRA_F16: return merge_states_d<TI, __half>(D, oa, la, ob, lb, n, out, lo, st);
    default: return merge_states_d<TI, __nv_bfloat16>(D, oa, la, ob, lb, n, out, lo, st);
  }
}
template <typename TO, int D>
bsra_status merge_many_t(const float* op, const float* lp, int P, int64_t n, void* out, float* lo, cudaStream_t st) {
  if (n == 0) return BSRA_OK;
  const int grid = (int)std::min<int64_t>((n + 7) / 8, 148 * 16);  // grid-stride loop: any size works
  bsra::merge_many_kernel<TO, D><<<grid, 256, 0, st>>>(op, lp, P, n, static_cast<TO*>(out), lo);
  CUDA_TRY(cudaGetLastError());
  return BSRA_OK;
}
}  // namespace

bsra_status bsra_merge_states(const void* o_a, const float* lse_a, const void* o_b, const float* lse_b,
                              bsra_dtype in_dtype, int64_t rows, int32_t heads, int32_t head_dim, void* o_out,
                              bsra_dtype out_dtype, float* lse_out, void* stream) {
  if (head_dim != 64 && head_dim != 128) return fail(BSRA_EUNSUPPORTED, "head_dim must be 64 or 128");
  if (rows < 0 || heads < 0) return fail(BSRA_EINVAL, "negative size");
  const int64_t n = rows * heads;
  if (n && (!o_a || !lse_a || !o_b || !lse_b || !o_out)) return fail(BSRA_EINVAL, "NULL pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (in_dtype) {
    case BSRA_F32: return merge_states_o<float>(out_dtype, head_dim, o_a, lse_a, o_b, lse_b, n, o_out, lse_out, st);
    case BSRA_F16: return merge_states_o<__half>(out_dtype, head_dim, o_a, lse_a, o_b, lse_b, n, o_out, lse_out, st);
    case BSRA_BF16:
      return merge_states_o<__nv_bfloat16>(out_dtype, head_dim, o_a, lse_a, o_b, lse_b, n, o_out, lse_out, st);
  }
  return fail(BSRA_EINVAL, "bad dtype");
}

bsra_status bsra_contract(bsra_engine* e, const float* o_extra, const float* lse_extra, void* o, int32_t o_dtype,
                          float* lse, void* stream) {
  if (!e) return fail(BSRA_EINVAL, "NULL engine");
  const bsra_config& c = e->cfg;
  if (!(c.flags & BSRA_FLAG_DEFER_CONTRACTION)) return fail(BSRA_EINVAL, "engine without BSRA_FLAG_DEFER_CONTRACTION");
  if (!e->have_deferred) return fail(BSRA_EINVAL, "no deferred run to contract");
  if (!o) return fail(BSRA_EINVAL, "NULL o");
  if ((o_extra == nullptr) != (lse_extra == nullptr)) return fail(BSRA_EINVAL, "o_extra and lse_extra: both or neither");
  if (o_extra && e->device_planned) return fail(BSRA_EUNSUPPORTED, "an extra state needs a host-built plan");
  if (o_extra && e->summary.n_slots != e->summary.n_items)
    return fail(BSRA_EUNSUPPORTED, "an extra state needs every item split (rows written through are final)");
  if (o_dtype != BSRA_F32 && o_dtype != BSRA_F16 && o_dtype != BSRA_BF16) return fail(BSRA_EINVAL, "bad o_dtype");
  bsra::AttnParams p = e->deferred;
  p.o = o;
  p.o_f32 = o_dtype == BSRA_F32;
  p.lse = lse;
  p.x_o = o_extra;
  p.x_lse = lse_extra;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int cgrid = contraction_grid(e);
  bsra_status s;
  const bool pdl = (c.flags & BSRA_FLAG_PDL) != 0;
  if (o_dtype == BSRA_F32) s = launch_contraction_d<float>(p, c.head_dim, cgrid, st, pdl);
  else if (o_dtype == BSRA_F16) s = launch_contraction_d<__half>(p, c.head_dim, cgrid, st, pdl);
  else s = launch_contraction_d<__nv_bfloat16>(p, c.head_dim, cgrid, st, pdl);
  return s;
}

bsra_status bsra_merge_many(const float* o_parts, const float* lse_parts, int32_t P, int64_t rows, int32_t heads,
                            int32_t head_dim, void* o_out, bsra_dtype out_dtype, float* lse_out, void* stream) {
  if (head_dim != 64 && head_dim != 128) return fail(BSRA_EUNSUPPORTED, "head_dim must be 64 or 128");
  if (P < 1 || rows < 0 || heads < 0) return fail(BSRA_EINVAL, "bad sizes");
  const int64_t n = rows * heads;
  if (n && (!o_parts || !lse_parts || !o_out)) return fail(BSRA_EINVAL, "NULL pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool d64 = head_dim == 64;
  switch (out_dtype) {
    case BSRA_F32:
      return d64 ? merge_many_t<float, 64>(o_parts, lse_parts, P, n, o_out, lse_out, st)
                 : merge_many_t<float, 128>(o_parts, lse_parts, P, n, o_out, lse_out, st);
    case BSRA_F16:
      return d64 ? merge_many_t<__half, 64>(o_parts, lse_parts, P, n, o_out, lse_out, st)
                 : merge_many_t<__half, 128>(o_parts, lse_parts, P, n, o_out, lse_out, st);
    case BSRA_BF16:
      return d64 ? merge_many_t<__nv_bfloat16, 64>(o_parts, lse_parts, P, n, o_out, lse_out, st)
                 : merge_many_t<__nv_bfloat16, 128>(o_parts, lse_parts, P, n, o_out, lse_out, st);
  }
  return fail(BSRA_EINVAL, "bad dtype");
}

bsra_status bsra_plan_export(const bsra_engine* e, int32_t from_device, int32_t* host_buf, size_t cap_words,
                             size_t* n_words, void* stream) {
  if (!e || !n_words) return fail(BSRA_EINVAL, "NULL argument");
  if (e->device_planned) {  // the image exists only on the device: its size from its header
    if (!from_device) return fail(BSRA_EINVAL, "device-built plan: export with from_device = 1");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t h[16];
    CUDA_TRY(cudaMemcpyAsync(h, e->ws + e->lay.off_plan, sizeof(h), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const size_t words = 16 + (size_t)(h[2] + 1) + 6 * (size_t)h[5] + (size_t)(h[6] + 1) + (size_t)h[7] +
                         3 * (size_t)h[6] + 4 * (size_t)h[8];
    *n_words = words;
    if (!host_buf) return BSRA_OK;
    if (cap_words < words) return fail(BSRA_ENOMEM, "buffer too small");
    CUDA_TRY(cudaMemcpyAsync(host_buf, e->ws + e->lay.off_plan, words * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return BSRA_OK;
  }
  *n_words = e->image.size();
  if (!host_buf) return BSRA_OK;
  if (cap_words < e->image.size()) return fail(BSRA_ENOMEM, "buffer too small");
  if (!from_device) {
    std::memcpy(host_buf, e->image.data(), e->image.size() * 4);
    return BSRA_OK;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CUDA_TRY(cudaMemcpyAsync(host_buf, e->ws + e->lay.off_plan, e->image.size() * 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return BSRA_OK;
}

bsra_status bsra_plan_stats(const bsra_engine* e, int64_t* cta_cost, int32_t cap, int64_t* makespan) {
  if (!e || !e->planned || e->image.empty()) return fail(BSRA_EINVAL, "no host plan (device-built plans: export them)");
  const int32_t* im = e->image.data();
  const int nc = im[2], T_q = im[3], n_items = im[5];
  const int64_t alpha = e->cfg.cost_alpha ? e->cfg.cost_alpha : 1, beta = e->cfg.cost_beta ? e->cfg.cost_beta : 1;
  const int32_t* ind = im + bsra::kHeaderWords;
  const int32_t* kb = ind + nc + 1 + 3 * n_items;
  const int32_t* ke = kb + n_items;
  int64_t mx = 0;
  for (int c = 0; c < nc; ++c) {
    int64_t s = 0;
    for (int it = ind[c]; it < ind[c + 1]; ++it) s += alpha * T_q + beta * (int64_t)(ke[it] - kb[it]);
    if (cta_cost && c < cap) cta_cost[c] = s;
    mx = std::max(mx, s);
  }
  if (makespan) *makespan = mx;
  return BSRA_OK;
}

