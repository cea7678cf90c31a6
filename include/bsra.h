/*
 * bsra.h — C ABI of libbsra.so: block-sparse-row (paged) attention for B200 (sm_100a).
 *
 * The hot path of FlashInfer (arXiv 2501.01005; /root/reference/PAPER.md, cited "P:<line>"):
 * attention of ragged query batches over a KV cache stored as a block-sparse-row matrix
 * (§3.1.1), scheduled by the load-balanced Algorithm 1 (§3.3.1), with
 * split-KV partial states combined by the attention-state operator ⊕ (§2.2).
 * The plan()/run() split follows the paper's inspector-executor interface (§3.4).
 *
 * Conventions (all functions):
 *   - every call returns bsra_status (0 = OK); no C++ exception crosses the ABI; on error a
 *     message is available from bsra_last_error() (thread-local, valid until the next call).
 *   - "host" pointers are ordinary CPU memory; "device" pointers are CUDA device memory on the
 *     engine's device. The caller owns every buffer it passes and every stream; nothing the
 *     caller passed is freed by the library. Streams are cudaStream_t passed as void*.
 *   - asynchronous CUDA failures surface as BSRA_ECUDA on a later call.
 *   - determinism: the same plan inputs give bitwise-identical outputs run to run.
 *   - one host thread per engine; engines are independent.
 */
#ifndef BSRA_H_
#define BSRA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BSRA_OK = 0,
  BSRA_EINVAL = 1,       /* malformed argument (NULL, bad indptr, unsupported combination) */
  BSRA_EBOUNDS = 2,      /* workload exceeds the bounds declared at engine creation */
  BSRA_EUNSUPPORTED = 3, /* valid but not implemented (e.g. head_dim not in {64,128}) */
  BSRA_ECUDA = 4,        /* CUDA runtime/driver error */
  BSRA_ENOMEM = 5,       /* host allocation failed or workspace too small */
  BSRA_ENCCL = 6         /* NCCL error (bsra_dist.h) */
} bsra_status;

/* BSRA_E4M3: OCP FP8 E4M3 ("E4M3FN": bias 7, no infinities, S.1111.111 = NaN, max 448), valid
 * only as bsra_config.kv_dtype — the fp8 KV cache of the paper's FP8-FP16 mixed-precision
 * attention, where "the query and output remain in fp16, while the KV-Cache is stored in fp8"
 * (App. F; R28). */
typedef enum { BSRA_F32 = 0, BSRA_F16 = 1, BSRA_BF16 = 2, BSRA_E4M3 = 3 } bsra_dtype;

/* LogitsMask. CAUSAL is right-aligned: query row r of a request with lengths
 * (l_qo, l_kv) sees token t iff t <= l_kv - l_qo + r (R4). CUSTOM: per request a
 * row-major l_qo x l_kv bit matrix, LSB-first within bytes, starting at bit offset
 * mask_bit_indptr[i] (R9). Masked pairs are skipped; a row that sees nothing gets
 * o = 0, lse = -inf (R3, R10). */
typedef enum { BSRA_MASK_NONE = 0, BSRA_MASK_CAUSAL = 1, BSRA_MASK_CUSTOM = 2 } bsra_mask;

/* Kernel family selection; AUTO picks the tcgen05 kernels where they apply (bf16/f16,
 * head_dim 128) and the CUDA-core kernel otherwise. SIMT forces the CUDA-core kernel
 * (cross-kernel tests). */
typedef enum { BSRA_KERNEL_AUTO = 0, BSRA_KERNEL_SIMT = 1, BSRA_KERNEL_TC = 2 } bsra_kernel;

typedef struct {
  int32_t num_qo_heads;      /* H_qo; H_qo % H_kv == 0; g = H_qo / H_kv                 */
  int32_t num_kv_heads;      /* H_kv                                                            */
  int32_t head_dim;          /* D in {64, 128}                                                  */
  int32_t page_size;         /* B_c >= 1 ("B_c is specified by KV-Cache management")   */
  bsra_dtype dtype;          /* dtype of q (and of k_pool, v_pool unless kv_dtype says otherwise) */
  bsra_dtype o_dtype;        /* = dtype, or BSRA_F32 (raw attention state for a later ⊕)      */
  bsra_mask mask;            /* fixed per engine                                                */
  int32_t max_batch;         /* scheduler-metadata bounds supplied up front (App. D.3) */
  int32_t max_total_qo_rows; /* bound on sum_i l_qo(i)                                          */
  int32_t num_ctas;          /* persistent grid size; 0 => 2 x #SM when T_q = 16, else #SM     */
  int32_t tile_set_mask;     /* allowed query tiles T_q: bit0=16, bit1=64, bit2=128, bit3=256
                                (256 = two 128-row MMA tiles sharing each K/V tile, R20);
                                0 => all */
  int32_t tile_q;            /* 0 => heuristic of §3.2.2; else forced T_q in {16,64,128,256} */
  int64_t cost_alpha;        /* Algorithm 1 cost(l_q, l_kv) = alpha*l_q + beta*l_kv     */
  int64_t cost_beta;         /*   0 => 1                                                        */
  int32_t kv_chunk_align;    /* chunk boundaries aligned to this many tokens; 0 => page_size  */
  int32_t kv_chunk_min;      /* floor for the chunk size L_kv; 0 => none                        */
  int32_t kernel;            /* bsra_kernel                                                     */
  int32_t flags;             /* BSRA_FLAG_* bits                                                */
  /* Attention variants (the paper's LogitsMask / LogitsTransform functors; compiled
   * in, no JIT). 0 = off. */
  int32_t sliding_window;    /* W > 0: row at position p = l_kv - l_qo + r also hides keys
                                t < p - W + 1 (W keys up to its own position; R26).
                                Algorithm 1 then starts each row's KV range at its window       */
  float logits_soft_cap;     /* c > 0: scaled logit s -> c * tanh(s / c) (R27)        */
  /* fp8 KV cache (App. F; R28). kv_dtype: 0 or == dtype => K/V in dtype;
   * BSRA_E4M3 => K/V pools hold one byte per element (dtype must be F16 or BF16; q and o stay in
   * dtype). Element values are k_scale * E4M3(byte) and v_scale * E4M3(byte): per-tensor
   * dequantisation scales (0 => 1), changeable per run with bsra_set_kv_scales. The kernels
   * dequantise exactly (every E4M3 value is exact in fp16 and bf16) and compute as for dtype.
   * Decode tiles (T_q = 16) dequantise inside the attention kernel. Prefill tiles (T_q >= 64)
   * on the tcgen05 path first gather the plan's tokens into a 16-bit copy in the caller's
   * WORKSPACE (one extra launch per run; 4 * max_total_kv_tokens * H_kv * head_dim bytes, sized
   * by bsra_workspace_bytes — the library never allocates device memory). */
  int32_t kv_dtype;
  float k_scale;
  float v_scale;
  /* ALiBi bias (a LogitsTransform, P:228 / P:554; R30): 1 => the scaled logit of key t
   * for query row r of qo head h gets + slope_h * (t - p), p = l_kv - l_qo + r, after the soft-cap;
   * slope_h = 2^(-8(h+1)/n) for h < n = 2^floor(log2 H_qo), else 2^(-4(2(h-n)+1)/n). 0 = off. */
  int32_t alibi;
  /* Bounds that fix launch choices independently of the plan, so one captured CUDA graph serves
   * every re-plan within them (App. D.1, "fixed offsets ... compatible with CUDAGraphs"):
   *   max_total_kv_tokens  bound on sum_i l_kv(i) (0 = none). Sizes the workspace region an E4M3
   *                        engine with prefill tiles gathers its 16-bit K/V copy into (such a
   *                        plan fails with EBOUNDS when it is 0 or exceeded), and is the token
   *                        extent of a contiguous-KV engine's K/V tensor maps under capture.
   *   max_qo_len           bound on any one request's l_qo (0 = none). When set, the decode
   *                        kernel's live fused columns are min(16, max_qo_len * g) for every plan
   *                        (plan() rejects a longer request with EBOUNDS); when 0 they follow each
   *                        plan and capture tracking (bsra_run) guards graphs against growth. */
  int32_t max_total_kv_tokens;
  int32_t max_qo_len;
  /* Fused RoPE (the paper's Query/KeyTransform, "fuse normalization, RoPE ... into the
   * attention kernel"; the StreamingLLM kernel of P:329-338; R31). rope_theta > 0 rotates
   * q and k inside the kernel before the logits: rotate-half pairs (i, i + D/2), frequency
   * theta_i = rope_theta^(-2i/D) / rope_scale, key t of a request at position t (its index in the
   * request's KV), query row r at l_kv - l_qo + r; the rotated q / k are rounded to `dtype` like
   * any query / key tensor (the MMA operand type). The K/V cache holds UN-rotated keys.
   * rope_scale 0 => 1. Not with an E4M3 KV cache (EUNSUPPORTED). Decode tiles (T_q = 16) rotate in
   * the tcgen05 decode kernel; other tiles run on the CUDA-core kernel. 0 = off. */
  float rope_theta;
  float rope_scale;
  int32_t reserved[2];       /* must be zero                                                    */
} bsra_config;

/* flags: BSRA_FLAG_PDL launches the tcgen05 kernels and the contraction kernel (bsra_run of
 * 64/128/256-row engines, bsra_contract) with programmatic dependent launch: a run() may start
 * streaming K/V while the previous kernel on the stream drains, and waits for it
 * (griddepcontrol.wait) before writing o / lse / workspace; the contraction kernel reads the
 * plan early and waits before reading the partial states. Only valid when the inputs of a
 * run() (q, pools, indices, mask) are NOT produced by the kernel immediately preceding it on
 * the stream — e.g. consecutive layers' attention captured back to back. */
#define BSRA_FLAG_PDL 1
/* flags: BSRA_FLAG_RAGGED_KV makes a contiguous-KV engine (the KV layout
 * the paper's App. B compares the page table against): K/V are ragged tensors
 * [sum l_kv, H_kv, D] indexed by kv_indptr, with no page table. Such an engine is planned with
 * bsra_plan_ragged and run with bsra_run_ragged, and requires page_size = 128 (the KV tile and
 * the default chunk alignment). */
#define BSRA_FLAG_RAGGED_KV 2
/* flags: BSRA_FLAG_BALANCE_CTAS makes bsra_plan run Algorithm 1 for every queue count c in
 * [num_ctas - num_ctas/8, num_ctas] and keep the plan with the smallest makespan under the
 * Algorithm-1 cost model (ties: larger c). The grid stays num_ctas (graphs stay valid): queues
 * c..num_ctas-1 are empty and those CTAs exit at once. With few long rows, L = ceil(sum/#CTA)
 * can leave a ragged last chunk per row (configs[4]: 4.6 chunks per row at 148 CTAs, makespan
 * 1.25x the mean; 144 queues give exactly 4.0). Costs ~c Algorithm-1 runs of host time per
 * plan, so it is off by default. */
#define BSRA_FLAG_BALANCE_CTAS 4
/* flags: BSRA_FLAG_CP_GATHER makes the tcgen05 decode kernel gather K/V token ROWS for every page
 * size, instead of one TMA box per (page, 64-column half): TMA tile::gather4 (4 rows of the pool
 * viewed as a 2-D [rows, head_dim] tensor per instruction) when K and V share strides that are
 * whole head_dim rows (NHD / HND pools), else 16-byte cp.async (4 token rows x 128 B per warp
 * instruction, zero-filled past the chunk). The row gather is always used where a TMA box cannot
 * tile the page (B_c < 8, or B_c neither dividing nor a multiple of 128; paged decode tiles); the
 * flag forces it elsewhere (the page-gather study of DESIGN.md). BSRA_FLAG_CP_ASYNC forces the
 * cp.async flavour of the row gather (A/B and tests). */
#define BSRA_FLAG_CP_GATHER 8
#define BSRA_FLAG_CP_ASYNC 16
/* flags: BSRA_FLAG_DEFER_CONTRACTION (engines whose tiles can exceed 16 rows, i.e. whose split
 * rows are merged by the separate contraction kernel): bsra_run launches only the attention
 * kernel; the split rows' partial states stay in the workspace until bsra_contract folds them.
 * This lets the contraction of one format fold a second format's state in the same pass
 * (composable formats: prefix ⊕ suffix). */
#define BSRA_FLAG_DEFER_CONTRACTION 32

typedef struct bsra_engine bsra_engine;

/* Library version (major*10000 + minor*100 + patch). */
int32_t bsra_version(void);

/* Number of SMs of a device (148 on B200); used for the num_ctas default (App. D.3). */
bsra_status bsra_num_sms(int32_t device, int32_t* out);

/* Bytes of device workspace an engine with this config needs (App. D.3):
 * a plan section sized from max_batch / max_total_qo_rows / num_ctas, and a partial-output
 * section of 2 x num_ctas tiles x T_q_max x (D + 1) fp32 words (the paper's bound taken per
 * KV-head tile, R19), plus arrival counters. Offsets are fixed for the engine's
 * lifetime so a CUDA graph can capture run() (App. D.1). Host-only, no CUDA calls if
 * cfg->num_ctas > 0. */
bsra_status bsra_workspace_bytes(const bsra_config* cfg, int32_t device, size_t* device_bytes);

/* Create an engine on `device` over a caller-allocated device workspace of ws_bytes
 * (>= bsra_workspace_bytes, 256-byte aligned). The engine owns a pinned host staging buffer
 * (App. D) and a host copy of the current plan. No device launches. */
bsra_status bsra_engine_create(const bsra_config* cfg, int32_t device, void* d_workspace, size_t ws_bytes,
                               bsra_engine** out);
void bsra_engine_destroy(bsra_engine* e);

/* Inspector: builds the load-balanced plan (Algorithm 1) from HOST arrays and
 * enqueues its upload (pinned staging -> fixed workspace section) on `stream`. Not CUDA-graph
 * capturable. One plan serves any number of run() calls with the same lengths.
 *   qo_indptr        [batch+1] host int32; qo_indptr[0] = 0; nondecreasing (ragged q/o)
 *   kv_page_indptr   [batch+1] host int32; kv_page_indptr[0] = 0; nondecreasing (BSR indptr)
 *   kv_last_page_len [batch]   host int32; in [1, page_size] when request i has pages
 *   sm_scale         logits scale (R1); <= 0 => 1/sqrt(head_dim)
 * Errors: EINVAL (malformed arrays), EBOUNDS (batch / rows beyond the declared bounds). */
bsra_status bsra_plan(bsra_engine* e, int32_t batch, const int32_t* qo_indptr, const int32_t* kv_page_indptr,
                      const int32_t* kv_last_page_len, float sm_scale, void* stream);

/* Executor: device pointers only; no allocation and no host synchronisation, so it is
 * CUDA-graph capturable. Uses the most recent plan of `e` in stream order.
 * Graph capture: a run() enqueued on a capturing stream bakes the plan's launch choices (query
 * tile T_q and kernel, the decode kernel's live columns, the fp8 gather pass, tensor-map extents)
 * into the graph. The engine records them, and every later bsra_plan / bsra_plan_ragged whose
 * plan a replay could not run correctly fails with BSRA_EBOUNDS and keeps the previous plan —
 * until bsra_graph_release(e) says those graphs are gone. Under capture the q tensor map spans
 * max_total_qo_rows rows, so the q buffer of a captured run must hold max_total_qo_rows rows
 * (contiguous KV: k / v must hold max_total_kv_tokens rows when that bound is set).
 *   q                [sum l_qo, H_qo, D] device, contiguous, cfg->dtype
 *   k_pool, v_pool   device pools; element (page p, slot s, kv head h, dim d) lives at
 *                    p*strides[0] + s*strides[1] + h*strides[2] + d  (strides in ELEMENTS, host
 *                    int64[3]; dim stride 1). Default NHD: [pages, page_size, H_kv, D].
 *                    Base addresses and strides must be 16-byte aligned. With kv_dtype =
 *                    BSRA_E4M3 the pools hold bytes (strides still in elements = bytes).
 *   kv_page_indices  [nnz] device int32: BSR `indices` (page ids); not validated (caller contract)
 *   custom_mask      MASK_CUSTOM: device uint8 bits (see bsra_mask); else NULL
 *   mask_bit_indptr  MASK_CUSTOM: device int64 [batch+1] bit offsets; else NULL
 *   o                [sum l_qo, H_qo, D] device, cfg->o_dtype, 32-byte aligned (the kernels
 *                    write whole 32-byte sectors of a row with 256-bit stores)
 *   lse              [sum l_qo, H_qo] device fp32, natural log (R2); NULL => not written
 * batch = 0 (or no rows) is a no-op that still launches the fixed kernels (graph stability). */
bsra_status bsra_run(bsra_engine* e, const void* q, const void* k_pool, const void* v_pool,
                     const int64_t* k_strides, const int64_t* v_strides, const int32_t* kv_page_indices,
                     const uint8_t* custom_mask, const int64_t* mask_bit_indptr, void* o, float* lse,
                     void* stream);

/* Contraction stage of the last bsra_run of a BSRA_FLAG_DEFER_CONTRACTION engine,
 * enqueued on `stream` (stream order after that run): every merge list of the current plan is
 * folded with ⊕ in plan order (R17) into o / lse (layout as bsra_run's o / lse; o in `o_dtype`,
 * BSRA_F32 / BSRA_F16 / BSRA_BF16, which may differ from the engine's o_dtype). With
 * o_extra / lse_extra (DEVICE fp32 [total_qo_rows, H_qo, head_dim] / [total_qo_rows, H_qo], the
 * layout of o) each folded row is further ⊕-combined with the extra state of the same output row,
 * in the same closed form (the composable formats' prefix ⊕ suffix). Rows the run
 * wrote through (unsplit items, App. D.2) are not touched, so an extra state requires a plan in
 * which every item is split (bsra_plan_stats / the image: n_slots == n_items): BSRA_EUNSUPPORTED
 * otherwise. o_extra / lse_extra: both or neither. A new plan cancels the pending contraction (the
 * next bsra_contract needs a run of that plan first). May be captured in a CUDA graph with the run.
 * Errors: EINVAL (no deferred run, flag not set, NULL o, bad o_dtype), EUNSUPPORTED. */
bsra_status bsra_contract(bsra_engine* e, const float* o_extra, const float* lse_extra, void* o, int32_t o_dtype,
                          float* lse, void* stream);

/* Device-side inspector (the paper's future work, "move the scheduler to device"): one
 * kernel builds, from DEVICE BSR arrays, the same plan image bsra_plan builds on the host (bit for
 * bit: same Algorithm 1, same tie-breaks), enqueued on `stream` — so a step's plan can be captured
 * in a CUDA graph with its run() calls and needs no host round trip.
 *   batch                  requests (host int, <= max_batch)
 *   d_qo_indptr, d_kv_page_indptr [batch+1], d_kv_last_page_len [batch]: DEVICE int32, read when
 *                          the kernel runs (stream order)
 * Requirements (the host must know the launch choices without the plan): paged engine, a fixed
 * tile (cfg.tile_q), cfg.max_qo_len for decode tiles, no BSRA_FLAG_BALANCE_CTAS, no fp8 prefill
 * tiles, num_ctas <= 512, at most 16,384 rows and 16,384 work items; the q buffer of later runs
 * must hold max_total_qo_rows rows. Errors found on the device (malformed arrays, bounds, too
 * large) leave an empty plan — run() then writes nothing — and a code that
 * bsra_plan_device_status returns (1 malformed, 2 bounds, 3 too large).
 * Host errors: EINVAL, EUNSUPPORTED (requirements), EBOUNDS (batch > max_batch). */
bsra_status bsra_plan_device(bsra_engine* e, int32_t batch, const int32_t* d_qo_indptr,
                             const int32_t* d_kv_page_indptr, const int32_t* d_kv_last_page_len, float sm_scale,
                             void* stream);

/* Synchronises `stream` and returns the device planner's status code (0 = OK) for the current plan
 * (0 for host-built plans). */
bsra_status bsra_plan_device_status(bsra_engine* e, void* stream, int32_t* code);

/* Declares that every CUDA graph captured over run() calls of `e` has been destroyed (or will
 * be re-captured): clears the launch choices recorded at capture, so the next plan may change
 * them. Host only. Errors: EINVAL (NULL engine). */
bsra_status bsra_graph_release(bsra_engine* e);

/* Dequantisation scales of an fp8 KV cache for subsequent run() calls on `e` (e.g. per layer);
 * 0 => 1. A captured graph keeps the scales of the run() it captured. Host only.
 * Errors: EINVAL (NULL engine, negative or non-finite scale). */
bsra_status bsra_set_kv_scales(bsra_engine* e, float k_scale, float v_scale);

/* Contiguous-KV inspector (engine created with BSRA_FLAG_RAGGED_KV): as bsra_plan, with the KV
 * lengths given by a ragged indptr instead of a page table.
 *   qo_indptr  [batch+1] host int32; [0] = 0; nondecreasing
 *   kv_indptr  [batch+1] host int32; [0] = 0; nondecreasing; request i's keys are rows
 *              kv_indptr[i] .. kv_indptr[i+1]-1 of k / v
 * Errors: EINVAL (malformed arrays, paged engine), EBOUNDS (bounds). */
bsra_status bsra_plan_ragged(bsra_engine* e, int32_t batch, const int32_t* qo_indptr, const int32_t* kv_indptr,
                             float sm_scale, void* stream);

/* Contiguous-KV executor: as bsra_run, with
 *   k, v       [kv_indptr[batch], H_kv, D] device, cfg->dtype; row t at t*strides[0], head h at
 *              h*strides[1] (ELEMENTS, host int64[2]; dim stride 1); base 16-byte aligned, strides
 *              16-byte multiples. Tiles are read with one TMA box per 128 tokens at a token
 *              coordinate (no gather); the tensor map's extent is kv_indptr[batch], so the last
 *              tile never reads past k / v.
 * q, custom_mask, mask_bit_indptr, o, lse, stream: as bsra_run. Graph-capturable. */
bsra_status bsra_run_ragged(bsra_engine* e, const void* q, const void* k, const void* v, const int64_t* k_strides,
                            const int64_t* v_strides, const uint8_t* custom_mask, const int64_t* mask_bit_indptr,
                            void* o, float* lse, void* stream);

/* ⊕ of two attention-state tensors, max-shifted, fp32 arithmetic; the empty state
 * (o = 0, lse = -inf) is the identity. rows x heads states of head_dim values each.
 *   o_a, o_b [rows, heads, D] device in in_dtype; lse_a, lse_b [rows, heads] device fp32
 *   o_out [rows, heads, D] device in out_dtype; lse_out fp32 or NULL. In place allowed. */
bsra_status bsra_merge_states(const void* o_a, const float* lse_a, const void* o_b, const float* lse_b,
                              bsra_dtype in_dtype, int64_t rows, int32_t heads, int32_t head_dim, void* o_out,
                              bsra_dtype out_dtype, float* lse_out, void* stream);

/* Left fold of ⊕ over P parts in part order: o_parts fp32 [P, rows, heads, D] and
 * lse_parts fp32 [P, rows, heads] (device) -> o_out (out_dtype), lse_out (fp32 or NULL). */
bsra_status bsra_merge_many(const float* o_parts, const float* lse_parts, int32_t P, int64_t rows,
                            int32_t heads, int32_t head_dim, void* o_out, bsra_dtype out_dtype, float* lse_out,
                            void* stream);

/* Host-only Algorithm 1: the plan image bsra_plan would build for this config and lengths with
 * `num_ctas` CTAs (no engine, no CUDA). Used for the bit-exact scheduler tests. */
bsra_status bsra_plan_host(const bsra_config* cfg, int32_t num_ctas, int32_t batch, const int32_t* qo_indptr,
                           const int32_t* kv_page_indptr, const int32_t* kv_last_page_len, int32_t* image,
                           size_t cap_words, size_t* n_words);

/* Copy of the engine's current plan image: host copy (from_device = 0) or read back from the
 * device workspace section after synchronising `stream` (from_device = 1). */
bsra_status bsra_plan_export(const bsra_engine* e, int32_t from_device, int32_t* host_buf, size_t cap_words,
                             size_t* n_words, void* stream);

/* Per-CTA cost of the current plan under the Algorithm-1 cost model, and its makespan. */
bsra_status bsra_plan_stats(const bsra_engine* e, int64_t* cta_cost, int32_t cap, int64_t* makespan);

/* Kernels launched by the most recent bsra_run (for launch-count reporting). */
int32_t bsra_last_run_launches(const bsra_engine* e);

/* Name of the attention kernel family the current plan selected ("simt", "tc_decode", "tc_prefill"). */
const char* bsra_selected_kernel(const bsra_engine* e);

const char* bsra_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BSRA_H_ */
