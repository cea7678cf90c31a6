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

/* Message of the last failing bsra_dist_* call on this thread (NCCL / dlopen errors). */
const char* bsra_dist_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* BSRA_DIST_H_ */
