/*
 * bsra_dist.h — cross-GPU combination of attention states for sequence-split long-context
 * decode (BASELINE configs[4]). Part of libbsra.so.
 *
 * The KV of each request is split along the sequence across P ranks; every rank runs the
 * paged attention of its shard (bsra_run with o_dtype = F32, lse requested) and the P partial
 * states (o, lse) are combined with the attention-state operator ⊕ (§2.2: "⊕ is
 * associative and commutative ... Ring-Attention and Flash-Decoding utilize this property").
 * The exchange is an NCCL all-gather of the fp32 states over NVLink/NVSwitch, followed on every
 * rank by a left fold of ⊕ in rank order, so all ranks hold bitwise-identical o and lse.
 *
 * NCCL is loaded at run time (dlopen "libnccl.so.2", or $BSRA_NCCL_PATH), so libbsra.so itself
 * has no link-time NCCL dependency. The NCCL unique id is shipped by the caller (e.g. through a
 * torch.distributed process group); the library owns the communicator.
 */
#ifndef BSRA_DIST_H_
#define BSRA_DIST_H_

#include "bsra.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bsra_dist bsra_dist;

/* Rank 0 creates the 128-byte NCCL unique id (host buffer). BSRA_ENCCL if NCCL is unavailable. */
bsra_status bsra_dist_unique_id(uint8_t id[128]);

/* Collective over nranks processes: create the communicator on `device` (one process per GPU). */
bsra_status bsra_dist_create(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device, bsra_dist** out);
void bsra_dist_destroy(bsra_dist* d);

/* Device bytes of gather scratch bsra_dist_allgather_merge needs: nranks * rows*heads*(D+1) fp32. */
bsra_status bsra_dist_scratch_bytes(const bsra_dist* d, int64_t rows, int32_t heads, int32_t head_dim, size_t* bytes);

/* All-gather of this rank's partial state and ⊕ over ranks 0..P-1 (in that order).
 *   o_local   [rows, heads, D] fp32 device; lse_local [rows, heads] fp32 device (natural log)
 *   scratch   >= bsra_dist_scratch_bytes, device, 256-byte aligned
 *   o_out     [rows, heads, D] device in out_dtype; lse_out [rows, heads] fp32 or NULL
 * Enqueued on `stream` (graph-capturable: NCCL + one merge kernel). Identical results on all ranks. */
bsra_status bsra_dist_allgather_merge(bsra_dist* d, const float* o_local, const float* lse_local, int64_t rows,
                                      int32_t heads, int32_t head_dim, void* scratch, void* o_out,
                                      bsra_dtype out_dtype, float* lse_out, void* stream);

/* Polls the communicator for an asynchronous NCCL failure (ncclCommGetAsyncError): BSRA_OK while
 * healthy or in progress, BSRA_ENCCL (message in bsra_dist_last_error) once NCCL reports an
 * error — e.g. a peer died or a network/NVLink fault. bsra_dist_allgather_merge polls it too. */
bsra_status bsra_dist_check(bsra_dist* d);

/* Sequence split of a BSR page table for long-context decode (BASELINE configs[4]; north_star
 * "very long contexts split along the sequence"): rank r of P owns the contiguous logical page
 * range [floor(r*n/P), floor((r+1)*n/P)) of every request, n = its page count. The shard is
 * itself a BSR table over the SAME physical pool (page ids are copied, not renumbered); its
 * last_page_len is the request's own on the rank that holds the request's final page and
 * page_size elsewhere (a rank with no page of request i gets l_kv = 0 there). ⊕ of the ranks'
 * states in rank order is the whole request's attention. Host only; no CUDA, no NCCL.
 *   kv_page_indptr [batch+1], kv_page_indices [kv_page_indptr[batch]], kv_last_page_len [batch]:
 *                  host int32, validated as in bsra_plan
 *   out_indptr [batch+1], out_last [batch]: host int32; out_indices: host int32, cap entries
 *                  (kv_page_indptr[batch] always suffices); may be NULL with cap = 0 to size it
 *   out_nnz        pages in this rank's shard
 * Errors: EINVAL (malformed table, rank not in [0, nranks)), ENOMEM (cap too small). */
bsra_status bsra_dist_shard_bsr(int32_t nranks, int32_t rank, int32_t batch, int32_t page_size,
                                const int32_t* kv_page_indptr, const int32_t* kv_page_indices,
                                const int32_t* kv_last_page_len, int32_t* out_indptr, int32_t* out_indices,
                                size_t cap, int32_t* out_last, int64_t* out_nnz);

/* KV-head partition for batched decode / prefill (north_star "requests and KV
 * heads sharded with no communication"): rank r of P owns kv heads [begin, end) with
 * begin = floor(r*H_kv/P), end = floor((r+1)*H_kv/P), and with them qo heads [begin*g, end*g)
 * (GQA groups never straddle ranks). Each rank runs its own engine with
 * num_kv_heads = end - begin over pools holding only those heads (or the full pools offset by
 * begin*head_dim elements with the full strides); its o is the head slice of the 1-GPU output,
 * so no collective is needed (output stays head-sharded, like tensor-parallel attention).
 * Host only. Errors: EINVAL (H_kv < 1, rank not in [0, nranks), NULL outputs). */
bsra_status bsra_dist_head_shard(int32_t num_kv_heads, int32_t nranks, int32_t rank, int32_t* kv_head_begin,
                                 int32_t* kv_head_end);

/* Message of the last failing bsra_dist_* call on this thread (NCCL / dlopen errors). */
const char* bsra_dist_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BSRA_DIST_H_ */
