// dist.cpp — bsra_dist_*: NCCL all-gather of partial attention states + ⊕ merge (include/bsra_dist.h).
// NCCL is resolved with dlopen at bsra_dist_create time (no link-time dependency).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/bsra_dist.h"

namespace {

// Minimal NCCL ABI (stable since NCCL 2.0): opaque comm, 128-byte unique id, enums as ints.
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // 0 = ncclSuccess
constexpr int kNcclFloat32 = 7;

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
};

thread_local std::string g_dist_err;

Nccl* nccl() {
  static Nccl n;
  static bool tried = false;
  if (tried) return n.h ? &n : nullptr;
  tried = true;
  const char* env = std::getenv("BSRA_NCCL_PATH");
  n.h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!n.h) {
    g_dist_err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return nullptr;
  }
#define LOAD(f) n.f = reinterpret_cast<decltype(n.f)>(dlsym(n.h, "nccl" #f))
  LOAD(GetUniqueId);
  LOAD(CommInitRank);
  LOAD(CommDestroy);
  LOAD(AllGather);
  LOAD(GroupStart);
  LOAD(GroupEnd);
  LOAD(GetErrorString);
  LOAD(CommGetAsyncError);
#undef LOAD
  if (!n.GetUniqueId || !n.CommInitRank || !n.AllGather || !n.GroupStart || !n.GroupEnd || !n.CommDestroy) {
    g_dist_err = "libnccl.so.2 lacks required symbols";
    n.h = nullptr;
    return nullptr;
  }
  return &n;
}

bsra_status nccl_fail(ncclResult_t r, const char* what) {
  Nccl* n = nccl();
  g_dist_err = std::string(what) + ": " + (n && n->GetErrorString ? n->GetErrorString(r) : "nccl error");
  return BSRA_ENCCL;
}

}  // namespace

struct bsra_dist {
  ncclComm_t comm = nullptr;
  int32_t nranks = 0, rank = 0, device = 0;
};

extern "C" const char* bsra_dist_last_error(void) { return g_dist_err.c_str(); }

bsra_status bsra_dist_unique_id(uint8_t id[128]) {
  if (!id) return BSRA_EINVAL;
  Nccl* n = nccl();
  if (!n) return BSRA_ENCCL;
  ncclUniqueId u;
  ncclResult_t r = n->GetUniqueId(&u);
  if (r) return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, u.internal, 128);
  return BSRA_OK;
}

bsra_status bsra_dist_create(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device, bsra_dist** out) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return BSRA_EINVAL;
  *out = nullptr;
  Nccl* n = nccl();
  if (!n) return BSRA_ENCCL;
  if (cudaSetDevice(device) != cudaSuccess) return BSRA_ECUDA;
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  auto* d = new bsra_dist();
  ncclResult_t r = n->CommInitRank(&d->comm, nranks, u, rank);
  if (r) {
    delete d;
    return nccl_fail(r, "ncclCommInitRank");
  }
  d->nranks = nranks;
  d->rank = rank;
  d->device = device;
  *out = d;
  return BSRA_OK;
}

void bsra_dist_destroy(bsra_dist* d) {
  if (!d) return;
  Nccl* n = nccl();
  if (n && d->comm) n->CommDestroy(d->comm);
  delete d;
}

static size_t align256(size_t x) { return (x + 255) / 256 * 256; }

bsra_status bsra_dist_scratch_bytes(const bsra_dist* d, int64_t rows, int32_t heads, int32_t head_dim, size_t* bytes) {
  if (!d || !bytes || rows < 0 || heads < 0 || head_dim <= 0) return BSRA_EINVAL;
  const size_t n = (size_t)rows * heads;
  *bytes = align256((size_t)d->nranks * n * head_dim * 4) + align256((size_t)d->nranks * n * 4);
  return BSRA_OK;
}

bsra_status bsra_dist_allgather_merge(bsra_dist* d, const float* o_local, const float* lse_local, int64_t rows,
                                      int32_t heads, int32_t head_dim, void* scratch, void* o_out,
                                      bsra_dtype out_dtype, float* lse_out, void* stream) {
  if (!d || !o_local || !lse_local || !scratch || !o_out) return BSRA_EINVAL;
  Nccl* n = nccl();
  if (!n) return BSRA_ENCCL;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t cnt = (size_t)rows * heads;
  float* go = static_cast<float*>(scratch);
  float* gl = reinterpret_cast<float*>(static_cast<uint8_t*>(scratch) + align256((size_t)d->nranks * cnt * head_dim * 4));
  bsra_status hs = bsra_dist_check(d);  // a communicator with a pending async error cannot be used
  if (hs) return hs;
  ncclResult_t r = n->GroupStart();
  if (!r) r = n->AllGather(o_local, go, cnt * head_dim, kNcclFloat32, d->comm, st);
  if (!r) r = n->AllGather(lse_local, gl, cnt, kNcclFloat32, d->comm, st);
  ncclResult_t r2 = n->GroupEnd();
  if (r) return nccl_fail(r, "ncclAllGather");
  if (r2) return nccl_fail(r2, "ncclGroupEnd");
  // ⊕ in rank order (identical on every rank): bsra_merge_many over [P, rows, heads, D]
  return bsra_merge_many(go, gl, d->nranks, rows, heads, head_dim, o_out, out_dtype, lse_out, stream);
}

bsra_status bsra_dist_check(bsra_dist* d) {
  if (!d) return BSRA_EINVAL;
  Nccl* n = nccl();
  if (!n) return BSRA_ENCCL;
  if (!n->CommGetAsyncError) return BSRA_OK;  // very old NCCL: nothing to poll
  ncclResult_t async = 0;
  ncclResult_t r = n->CommGetAsyncError(d->comm, &async);
  if (r) return nccl_fail(r, "ncclCommGetAsyncError");
  constexpr ncclResult_t kInProgress = 7;  // ncclInProgress (non-blocking communicators)
  if (async != 0 && async != kInProgress) return nccl_fail(async, "NCCL asynchronous error");
  return BSRA_OK;
}

bsra_status bsra_dist_shard_bsr(int32_t nranks, int32_t rank, int32_t batch, int32_t page_size,
                                const int32_t* kv_page_indptr, const int32_t* kv_page_indices,
                                const int32_t* kv_last_page_len, int32_t* out_indptr, int32_t* out_indices,
                                size_t cap, int32_t* out_last, int64_t* out_nnz) {
  if (nranks < 1 || rank < 0 || rank >= nranks || batch < 0 || page_size < 1 || !out_nnz) {
    g_dist_err = "bad nranks / rank / batch / page_size";
    return BSRA_EINVAL;
  }
  if (batch > 0 && (!kv_page_indptr || !kv_last_page_len || !out_indptr || !out_last)) {
    g_dist_err = "NULL array";
    return BSRA_EINVAL;
  }
  if (batch > 0 && kv_page_indptr[0] != 0) {
    g_dist_err = "kv_page_indptr[0] != 0";
    return BSRA_EINVAL;
  }
  int64_t nnz = 0;
  for (int32_t i = 0; i < batch; ++i) {  // validate and size
    const int64_t n = (int64_t)kv_page_indptr[i + 1] - kv_page_indptr[i];
    if (n < 0 || (n > 0 && (kv_last_page_len[i] < 1 || kv_last_page_len[i] > page_size))) {
      g_dist_err = "malformed BSR table at request " + std::to_string(i);
      return BSRA_EINVAL;
    }
    nnz += (rank + 1) * n / nranks - rank * n / nranks;
  }
  *out_nnz = nnz;
  if (!out_indices && cap == 0) {  // sizing call
    if (batch > 0) out_indptr[0] = 0;
    return BSRA_OK;
  }
  if ((int64_t)cap < nnz || (nnz > 0 && !out_indices)) {
    g_dist_err = "out_indices capacity too small";
    return BSRA_ENOMEM;
  }
  if (nnz > 0 && !kv_page_indices) {
    g_dist_err = "NULL kv_page_indices";
    return BSRA_EINVAL;
  }
  int64_t w = 0;
  if (batch > 0) out_indptr[0] = 0;
  for (int32_t i = 0; i < batch; ++i) {
    const int64_t n = (int64_t)kv_page_indptr[i + 1] - kv_page_indptr[i];
    const int64_t a = rank * n / nranks, b = (rank + 1) * n / nranks;
    for (int64_t j = a; j < b; ++j) out_indices[w++] = kv_page_indices[kv_page_indptr[i] + j];
    out_indptr[i + 1] = (int32_t)w;
    out_last[i] = (b == n && b > a) ? kv_last_page_len[i] : page_size;
  }
  return BSRA_OK;
}

bsra_status bsra_dist_head_shard(int32_t num_kv_heads, int32_t nranks, int32_t rank, int32_t* kv_head_begin,
                                 int32_t* kv_head_end) {
  if (num_kv_heads < 1 || nranks < 1 || rank < 0 || rank >= nranks || !kv_head_begin || !kv_head_end) {
    g_dist_err = "bad num_kv_heads / nranks / rank, or NULL output";
    return BSRA_EINVAL;
  }
  *kv_head_begin = (int32_t)((int64_t)rank * num_kv_heads / nranks);
  *kv_head_end = (int32_t)((int64_t)(rank + 1) * num_kv_heads / nranks);
  return BSRA_OK;
}
