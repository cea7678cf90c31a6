"""bsra — block-sparse-row (paged) attention for B200: thin Python binding of libbsra.so.

Argument marshalling only (ctypes over the C ABI in include/bsra.h): every step of the hot
path runs in libbsra.so (host scheduler + sm_100a kernels). There is no CPU or PyTorch
fallback: if libbsra.so is missing or a call fails, an exception is raised.

PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BSRA_LIB") or os.path.join(_HERE, "libbsra.so")  # override: A/B builds

F32, F16, BF16, E4M3 = 0, 1, 2, 3
MASK = {"none": 0, "causal": 1, "custom": 2}
DTYPE = {"f32": F32, "f16": F16, "bf16": BF16, "e4m3": E4M3}
TORCH_DTYPE = {F32: torch.float32, F16: torch.float16, BF16: torch.bfloat16, E4M3: torch.float8_e4m3fn}
KERNEL = {"auto": 0, "simt": 1, "tc": 2}
TILE_BIT = {16: 1, 64: 2, 128: 4, 256: 8}


class BsraError(RuntimeError):
    pass


class Config(ctypes.Structure):
    _fields_ = [("num_qo_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("dtype", ctypes.c_int32), ("o_dtype", ctypes.c_int32),
                ("mask", ctypes.c_int32), ("max_batch", ctypes.c_int32), ("max_total_qo_rows", ctypes.c_int32),
                ("num_ctas", ctypes.c_int32), ("tile_set_mask", ctypes.c_int32), ("tile_q", ctypes.c_int32),
                ("cost_alpha", ctypes.c_int64), ("cost_beta", ctypes.c_int64), ("kv_chunk_align", ctypes.c_int32),
                ("kv_chunk_min", ctypes.c_int32), ("kernel", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("sliding_window", ctypes.c_int32), ("logits_soft_cap", ctypes.c_float),
                ("kv_dtype", ctypes.c_int32), ("k_scale", ctypes.c_float), ("v_scale", ctypes.c_float),
                ("alibi", ctypes.c_int32), ("max_total_kv_tokens", ctypes.c_int32), ("max_qo_len", ctypes.c_int32),
                ("rope_theta", ctypes.c_float), ("rope_scale", ctypes.c_float), ("reserved", ctypes.c_int32 * 2)]


FLAG_PDL = 1  # BSRA_FLAG_PDL (include/bsra.h)
FLAG_RAGGED_KV = 2  # BSRA_FLAG_RAGGED_KV: contiguous (ragged) K/V, no page table
FLAG_BALANCE_CTAS = 4  # BSRA_FLAG_BALANCE_CTAS: plan with the queue count that minimises the makespan
FLAG_CP_GATHER = 8  # BSRA_FLAG_CP_GATHER: decode kernel gathers K/V rows (TMA gather4 or cp.async)
FLAG_CP_ASYNC = 16  # BSRA_FLAG_CP_ASYNC: ... with 16-byte cp.async
FLAG_DEFER_CONTRACTION = 32  # BSRA_FLAG_DEFER_CONTRACTION: run() leaves split rows to bsra_contract


_lib = None
EXPORTS = ["bsra_version", "bsra_num_sms", "bsra_workspace_bytes", "bsra_engine_create", "bsra_engine_destroy",
           "bsra_plan", "bsra_run", "bsra_contract", "bsra_graph_release", "bsra_plan_device", "bsra_plan_device_status", "bsra_set_kv_scales", "bsra_plan_ragged", "bsra_run_ragged", "bsra_merge_states", "bsra_merge_many",
           "bsra_plan_host", "bsra_plan_export",
           "bsra_plan_stats", "bsra_last_run_launches", "bsra_selected_kernel", "bsra_last_error",
           "bsra_dist_unique_id", "bsra_dist_create", "bsra_dist_destroy", "bsra_dist_scratch_bytes",
           "bsra_dist_allgather_merge", "bsra_dist_check", "bsra_dist_shard_bsr", "bsra_dist_head_shard",
           "bsra_dist_last_error"]


def lib():
    """Load libbsra.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BsraError(f"{LIB_PATH} not built: run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        CP = ctypes.POINTER(Config)
        sig = {
            "bsra_version": (I32, []),
            "bsra_num_sms": (I32, [I32, P]),
            "bsra_workspace_bytes": (I32, [CP, I32, ctypes.POINTER(SZ)]),
            "bsra_engine_create": (I32, [CP, I32, P, SZ, ctypes.POINTER(P)]),
            "bsra_engine_destroy": (None, [P]),
            "bsra_plan": (I32, [P, I32, P, P, P, ctypes.c_float, P]),
            "bsra_run": (I32, [P, P, P, P, P, P, P, P, P, P, P, P]),
            "bsra_contract": (I32, [P, P, P, P, I32, P, P]),
            "bsra_set_kv_scales": (I32, [P, ctypes.c_float, ctypes.c_float]),
            "bsra_graph_release": (I32, [P]),
            "bsra_plan_device": (I32, [P, I32, P, P, P, ctypes.c_float, P]),
            "bsra_plan_device_status": (I32, [P, P, ctypes.POINTER(I32)]),
            "bsra_plan_ragged": (I32, [P, I32, P, P, ctypes.c_float, P]),
            "bsra_run_ragged": (I32, [P, P, P, P, P, P, P, P, P, P, P]),
            "bsra_merge_states": (I32, [P, P, P, P, I32, I64, I32, I32, P, I32, P, P]),
            "bsra_merge_many": (I32, [P, P, I32, I64, I32, I32, P, I32, P, P]),
            "bsra_plan_host": (I32, [CP, I32, I32, P, P, P, P, SZ, ctypes.POINTER(SZ)]),
            "bsra_plan_export": (I32, [P, I32, P, SZ, ctypes.POINTER(SZ), P]),
            "bsra_plan_stats": (I32, [P, P, I32, P]),
            "bsra_last_run_launches": (I32, [P]),
            "bsra_selected_kernel": (ctypes.c_char_p, [P]),
            "bsra_last_error": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise BsraError(f"bsra status {rc}: {lib().bsra_last_error().decode()}")


def _p(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def make_config(*, H_qo, H_kv, D, page_size, dtype="bf16", o_dtype=None, mask="none", max_batch=1,
                max_total_qo_rows=1, num_ctas=0, tile_set=(16, 64, 128, 256), tile_q=0, alpha=1, beta=1,
                kv_chunk_align=0, kv_chunk_min=0, kernel="auto", pdl=False, ragged_kv=False, window=0,
                soft_cap=0.0, kv_dtype=None, k_scale=0.0, v_scale=0.0, alibi=False, balance_ctas=False,
                max_total_kv_tokens=0, max_qo_len=0, rope_theta=0.0, rope_scale=0.0, cp_gather=False, cp_async=False,
                defer_contraction=False) -> Config:
    """window: sliding window W (0 = off, R26); soft_cap: logits soft-cap c (0 = off, R27);
    kv_dtype "e4m3": fp8 KV cache with per-tensor scales k_scale / v_scale (0 = 1; R28);
    max_total_kv_tokens / max_qo_len: engine bounds (include/bsra.h)."""
    c = Config()
    c.max_total_kv_tokens, c.max_qo_len = int(max_total_kv_tokens), int(max_qo_len)
    c.rope_theta, c.rope_scale = float(rope_theta), float(rope_scale)
    if kv_dtype:
        c.kv_dtype = DTYPE[kv_dtype] if isinstance(kv_dtype, str) else kv_dtype
    c.k_scale, c.v_scale = float(k_scale), float(v_scale)
    c.alibi = 1 if alibi else 0
    c.sliding_window, c.logits_soft_cap = int(window), float(soft_cap)
    c.flags = ((FLAG_PDL if pdl else 0) | (FLAG_RAGGED_KV if ragged_kv else 0) | (FLAG_BALANCE_CTAS if balance_ctas else 0)
               | (FLAG_CP_GATHER if cp_gather else 0) | (FLAG_CP_ASYNC if cp_async else 0)
               | (FLAG_DEFER_CONTRACTION if defer_contraction else 0))
    c.num_qo_heads, c.num_kv_heads, c.head_dim, c.page_size = H_qo, H_kv, D, page_size
    c.dtype = DTYPE[dtype] if isinstance(dtype, str) else dtype
    od = o_dtype if o_dtype is not None else dtype
    c.o_dtype = DTYPE[od] if isinstance(od, str) else od
    c.mask = MASK[mask] if isinstance(mask, str) else mask
    c.max_batch, c.max_total_qo_rows, c.num_ctas = max_batch, max_total_qo_rows, num_ctas
    c.tile_set_mask = sum(TILE_BIT[t] for t in tile_set)
    c.tile_q, c.cost_alpha, c.cost_beta = tile_q, alpha, beta
    c.kv_chunk_align, c.kv_chunk_min = kv_chunk_align, kv_chunk_min
    c.kernel = KERNEL[kernel] if isinstance(kernel, str) else kernel
    return c


def num_sms(device: int = 0) -> int:
    out = ctypes.c_int32()
    _check(lib().bsra_num_sms(device, ctypes.byref(out)))
    return out.value


def plan_host(cfg: Config, num_ctas: int, qo_indptr, kv_page_indptr, kv_last_page_len) -> np.ndarray:
    """Algorithm-1 plan image computed by the C++ scheduler (host only, no CUDA)."""
    qi, ki, kl = _i32(qo_indptr), _i32(kv_page_indptr), _i32(kv_last_page_len)
    n = ctypes.c_size_t()
    L = lib()
    _check(L.bsra_plan_host(ctypes.byref(cfg), num_ctas, len(qi) - 1, _p(qi), _p(ki), _p(kl), None, 0,
                            ctypes.byref(n)))
    out = np.zeros(n.value, np.int32)
    _check(L.bsra_plan_host(ctypes.byref(cfg), num_ctas, len(qi) - 1, _p(qi), _p(ki), _p(kl), _p(out), n.value,
                            ctypes.byref(n)))
    return out


class Engine:
    """One attention wrapper: fixed variant/task info + a device workspace it sizes."""

    def __init__(self, cfg: Config, device: int = 0):
        self.cfg = cfg
        self.device = device
        L = lib()
        nbytes = ctypes.c_size_t()
        _check(L.bsra_workspace_bytes(ctypes.byref(cfg), device, ctypes.byref(nbytes)))
        self.workspace = torch.empty(max(256, nbytes.value), dtype=torch.uint8, device=f"cuda:{device}")
        h = ctypes.c_void_p()
        _check(L.bsra_engine_create(ctypes.byref(cfg), device, self.workspace.data_ptr(), self.workspace.numel(),
                                    ctypes.byref(h)))
        self._h = h
        self._keep = []

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().bsra_engine_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream(stream):
        if stream is None:
            return torch.cuda.current_stream().cuda_stream
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)

    def plan(self, qo_indptr, kv_page_indptr, kv_last_page_len, sm_scale: float = 0.0, stream=None):
        qi, ki, kl = _i32(qo_indptr), _i32(kv_page_indptr), _i32(kv_last_page_len)
        self._keep = [qi, ki, kl]
        _check(lib().bsra_plan(self._h, len(qi) - 1, _p(qi), _p(ki), _p(kl), float(sm_scale), self._stream(stream)))

    def run(self, q, k_pool, v_pool, k_strides, v_strides, kv_page_indices, o, lse=None, custom_mask=None,
            mask_bit_indptr=None, stream=None):
        ks = (ctypes.c_int64 * 3)(*[int(x) for x in k_strides])
        vs = (ctypes.c_int64 * 3)(*[int(x) for x in v_strides])
        _check(lib().bsra_run(self._h, _p(q), _p(k_pool), _p(v_pool), ctypes.cast(ks, ctypes.c_void_p),
                              ctypes.cast(vs, ctypes.c_void_p), _p(kv_page_indices), _p(custom_mask),
                              _p(mask_bit_indptr), _p(o), _p(lse), self._stream(stream)))

    def plan_device(self, batch, qo_indptr, kv_page_indptr, kv_last_page_len, sm_scale: float = 0.0, stream=None):
        """Device-side Algorithm 1 (bsra_plan_device): the arrays are device int32 tensors."""
        _check(lib().bsra_plan_device(self._h, int(batch), _p(qo_indptr), _p(kv_page_indptr), _p(kv_last_page_len),
                                      float(sm_scale), self._stream(stream)))

    def plan_device_status(self, stream=None) -> int:
        code = ctypes.c_int32()
        _check(lib().bsra_plan_device_status(self._h, self._stream(stream), ctypes.byref(code)))
        return code.value

    def graph_release(self):
        """Every CUDA graph captured over this engine's run() calls is gone (bsra_graph_release)."""
        _check(lib().bsra_graph_release(self._h))

    def set_kv_scales(self, k_scale: float, v_scale: float):
        """fp8 KV dequantisation scales for the following run() calls (0 = 1)."""
        _check(lib().bsra_set_kv_scales(self._h, float(k_scale), float(v_scale)))

    def plan_ragged(self, qo_indptr, kv_indptr, sm_scale: float = 0.0, stream=None):
        """Contiguous-KV inspector (engine made with ragged_kv=True): kv_indptr[batch+1] token offsets."""
        qi, ki = _i32(qo_indptr), _i32(kv_indptr)
        self._keep = [qi, ki]
        _check(lib().bsra_plan_ragged(self._h, len(qi) - 1, _p(qi), _p(ki), float(sm_scale), self._stream(stream)))

    def run_ragged(self, q, k, v, k_strides, v_strides, o, lse=None, custom_mask=None, mask_bit_indptr=None,
                   stream=None):
        """Contiguous-KV executor: k, v [N, H_kv, D]; strides (token, head) in elements."""
        ks = (ctypes.c_int64 * 2)(*[int(x) for x in k_strides])
        vs = (ctypes.c_int64 * 2)(*[int(x) for x in v_strides])
        _check(lib().bsra_run_ragged(self._h, _p(q), _p(k), _p(v), ctypes.cast(ks, ctypes.c_void_p),
                                     ctypes.cast(vs, ctypes.c_void_p), _p(custom_mask), _p(mask_bit_indptr), _p(o),
                                     _p(lse), self._stream(stream)))

    def contract(self, o, lse=None, o_extra=None, lse_extra=None, stream=None):
        """bsra_contract: fold the deferred run's merge lists into o / lse, each row ⊕ the extra
        state (o_extra fp32 [rows, H_qo, D], lse_extra [rows, H_qo]) when given."""
        inv = {v: k for k, v in TORCH_DTYPE.items()}
        _check(lib().bsra_contract(self._h, _p(o_extra), _p(lse_extra), _p(o), inv[o.dtype], _p(lse),
                                   self._stream(stream)))

    def export_plan(self, from_device=False, stream=None) -> np.ndarray:
        L = lib()
        n = ctypes.c_size_t()
        st = self._stream(stream) if from_device else None
        _check(L.bsra_plan_export(self._h, int(from_device), None, 0, ctypes.byref(n), st))
        out = np.zeros(n.value, np.int32)
        _check(L.bsra_plan_export(self._h, int(from_device), _p(out), n.value, ctypes.byref(n),
                                  self._stream(stream) if from_device else None))
        return out

    def plan_stats(self):
        nc = int(self.export_plan()[2]) if self.export_plan().size else 0
        costs = np.zeros(max(nc, 1), np.int64)
        mk = ctypes.c_int64()
        _check(lib().bsra_plan_stats(self._h, _p(costs), nc, ctypes.byref(mk)))
        return costs[:nc], mk.value

    def last_launches(self) -> int:
        return lib().bsra_last_run_launches(self._h)

    def selected_kernel(self) -> str:
        return lib().bsra_selected_kernel(self._h).decode()


def merge_states(o_a, lse_a, o_b, lse_b, o_out=None, lse_out=None, stream=None):
    """⊕ of two state tensors: o [rows, heads, D], lse [rows, heads] fp32."""
    rows, heads, D = o_a.shape
    out_dtype = o_out.dtype if o_out is not None else o_a.dtype
    if o_out is None:
        o_out = torch.empty_like(o_a)
    if lse_out is None:
        lse_out = torch.empty_like(lse_a)
    inv = {v: k for k, v in TORCH_DTYPE.items()}
    _check(lib().bsra_merge_states(_p(o_a), _p(lse_a), _p(o_b), _p(lse_b), inv[o_a.dtype], rows, heads, D,
                                   _p(o_out), inv[out_dtype], _p(lse_out), Engine._stream(stream)))
    return o_out, lse_out


def merge_many(o_parts, lse_parts, o_out, lse_out=None, stream=None):
    """Left fold of ⊕ over parts (fp32 [P, rows, heads, D] / [P, rows, heads])."""
    P, rows, heads, D = o_parts.shape
    inv = {v: k for k, v in TORCH_DTYPE.items()}
    _check(lib().bsra_merge_many(_p(o_parts), _p(lse_parts), P, rows, heads, D, _p(o_out), inv[o_out.dtype],
                                 _p(lse_out), Engine._stream(stream)))
    return o_out, lse_out


def sequence_shard(kv_page_indptr, kv_page_indices, kv_last_page_len, page_size, nranks, rank):
    """Sequence split of a BSR page table for long-context decode (BASELINE configs[4]): the
    shard rank `rank` of `nranks` owns (bsra_dist_shard_bsr, include/bsra_dist.h). Marshalling
    only; returns (kv_page_indptr, kv_page_indices, kv_last_page_len) of the shard."""
    kp, idx, last = _i32(kv_page_indptr), _i32(kv_page_indices), _i32(kv_last_page_len)
    B = len(kp) - 1
    L = lib()
    P = ctypes.c_void_p
    L.bsra_dist_shard_bsr.restype = ctypes.c_int32
    L.bsra_dist_shard_bsr.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P,
                                      ctypes.c_size_t, P, ctypes.POINTER(ctypes.c_int64)]
    out_ip = np.zeros(B + 1, np.int32)
    out_last = np.zeros(max(B, 0), np.int32)
    out_idx = np.zeros(max(1, idx.size), np.int32)
    nnz = ctypes.c_int64()
    rc = L.bsra_dist_shard_bsr(nranks, rank, B, page_size, _p(kp), _p(idx), _p(last), _p(out_ip), _p(out_idx),
                               out_idx.size, _p(out_last), ctypes.byref(nnz))
    if rc:
        raise BsraError(f"bsra_dist_shard_bsr: {rc}: {Dist.last_error()}")
    return out_ip, out_idx[:nnz.value].copy(), out_last


def head_shard(num_kv_heads: int, nranks: int, rank: int):
    """KV heads [begin, end) rank `rank` of `nranks` owns (bsra_dist_head_shard)."""
    L = lib()
    L.bsra_dist_head_shard.restype = ctypes.c_int32
    b, e = ctypes.c_int32(), ctypes.c_int32()
    rc = L.bsra_dist_head_shard(num_kv_heads, nranks, rank, ctypes.byref(b), ctypes.byref(e))
    if rc:
        raise BsraError(f"bsra_dist_head_shard: {rc}: {Dist.last_error()}")
    return b.value, e.value


class Dist:
    """NCCL communicator owned by libbsra (include/bsra_dist.h); the unique id travels through
    the caller's process group (torch.distributed is plumbing only)."""

    def __init__(self, nranks: int, rank: int, uid: bytes, device: int = 0):
        L = lib()
        L.bsra_dist_create.restype = ctypes.c_int32
        L.bsra_dist_create.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_char_p, ctypes.c_int32,
                                       ctypes.POINTER(ctypes.c_void_p)]
        h = ctypes.c_void_p()
        rc = L.bsra_dist_create(nranks, rank, uid, device, ctypes.byref(h))
        if rc:
            raise BsraError(f"bsra_dist_create: {rc}: {Dist.last_error()}")
        self._h, self.nranks, self.rank = h, nranks, rank

    @staticmethod
    def last_error() -> str:
        f = lib().bsra_dist_last_error
        f.restype = ctypes.c_char_p
        return f().decode()

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        rc = lib().bsra_dist_unique_id(buf)
        if rc:
            raise BsraError(f"bsra_dist_unique_id: {rc}: {Dist.last_error()}")
        return buf.raw

    def scratch(self, rows, heads, D, device):
        n = ctypes.c_size_t()
        L = lib()
        L.bsra_dist_scratch_bytes.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                              ctypes.POINTER(ctypes.c_size_t)]
        _check(L.bsra_dist_scratch_bytes(self._h, rows, heads, D, ctypes.byref(n)))
        return torch.empty(n.value, dtype=torch.uint8, device=device)

    def allgather_merge(self, o_local, lse_local, scratch, o_out, lse_out=None, stream=None):
        rows, heads, D = o_local.shape
        inv = {v: k for k, v in TORCH_DTYPE.items()}
        L = lib()
        P = ctypes.c_void_p
        L.bsra_dist_allgather_merge.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P, P,
                                                ctypes.c_int32, P, P]
        rc = L.bsra_dist_allgather_merge(self._h, _p(o_local), _p(lse_local), rows, heads, D, _p(scratch), _p(o_out),
                                         inv[o_out.dtype], _p(lse_out), Engine._stream(stream))
        if rc:
            raise BsraError(f"bsra_dist_allgather_merge: {rc}: {Dist.last_error()} {L.bsra_last_error().decode()}")
        return o_out, lse_out

    def check(self):
        """Raise if NCCL reported an asynchronous error on this communicator (bsra_dist_check)."""
        L = lib()
        L.bsra_dist_check.argtypes = [ctypes.c_void_p]
        rc = L.bsra_dist_check(self._h)
        if rc:
            raise BsraError(f"bsra_dist_check: {rc}: {Dist.last_error()}")

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().bsra_dist_destroy(self._h)
            self._h = ctypes.c_void_p()


class ComposableDecode:
    """Composable formats: the KV of n branches that share a prefix is
    described as two BSR matrices over one pool — a shared-prefix block read once for all n
    query rows (large B_r: one "request" with l_qo = n, tensor-core tile; with g = 4 and n = 64
    the 256 fused rows are one paired 256-row tile, so every prefix K/V tile staged in shared
    memory serves all branches) and per-branch suffix blocks (B_r = 1) — one engine ("wrapper")
    each; the two attention states are combined with ⊕. The prefix engine defers its contraction
    (BSRA_FLAG_DEFER_CONTRACTION): when every prefix item is split, one bsra_contract launch folds
    the prefix's partial states AND the suffix state into o (prefix ⊕ suffix in one pass);
    otherwise its contraction writes the prefix state and bsra_merge_states combines the two.

    concurrent: the two engines run at the same time on disjoint SM sets — the prefix engine's
    persistent grid takes `prefix_ctas` SMs (tensor-bound tiles), the suffix engine the other
    `suffix_ctas` (HBM-bound) — forked on a side stream and joined before the ⊕, so the prefix's
    tensor work overlaps the suffix's HBM streaming (the joint plan of SURVEY §8(f) NEXT-4 as two
    co-resident persistent grids). All launches are graph-capturable."""

    def __init__(self, *, H_qo, H_kv, D, page_size, n_branch, dtype="bf16", device=0, prefix_ctas=0,
                 suffix_ctas=0, kernel="auto", prefix_tiles=(64, 128, 256), balance=True, concurrent=False,
                 pdl=False, suffix_pdl=None, suffix_first=False):
        self.n, self.H_qo, self.D = n_branch, H_qo, D
        self.concurrent = concurrent
        self.suffix_first = suffix_first  # sequential order: suffix kernel, then prefix kernel
        self.prefix = Engine(make_config(H_qo=H_qo, H_kv=H_kv, D=D, page_size=page_size, dtype=dtype, o_dtype="f32",
                                         max_batch=1, max_total_qo_rows=n_branch, num_ctas=prefix_ctas,
                                         tile_set=prefix_tiles, kernel=kernel, balance_ctas=balance, pdl=pdl,
                                         defer_contraction=True), device)
        self.suffix = Engine(make_config(H_qo=H_qo, H_kv=H_kv, D=D, page_size=page_size, dtype=dtype, o_dtype="f32",
                                         max_batch=n_branch, max_total_qo_rows=n_branch, num_ctas=suffix_ctas,
                                         tile_q=16, kernel=kernel, max_qo_len=1,
                                         pdl=pdl if suffix_pdl is None else suffix_pdl), device)
        dev = f"cuda:{device}"
        self.o_p = torch.empty((n_branch, H_qo, D), device=dev)
        self.l_p = torch.empty((n_branch, H_qo), device=dev)
        self.o_s = torch.empty((n_branch, H_qo, D), device=dev)
        self.l_s = torch.empty((n_branch, H_qo), device=dev)
        self.side = torch.cuda.Stream(device=dev) if concurrent else None
        self.fold_suffix = False

    def plan(self, prefix: dict, suffix: dict, sm_scale=0.0, stream=None):
        self.prefix.plan(prefix["qo_indptr"], prefix["kv_page_indptr"], prefix["kv_last_page_len"], sm_scale, stream)
        self.suffix.plan(suffix["qo_indptr"], suffix["kv_page_indptr"], suffix["kv_last_page_len"], sm_scale, stream)
        img = self.prefix.export_plan()
        self.fold_suffix = bool(img.size) and int(img[5]) == int(img[7])  # every prefix item split

    def run(self, q, k_pool, v_pool, strides, prefix_indices, suffix_indices, o, lse=None, stream=None):
        st = stream if stream is not None else torch.cuda.current_stream()
        if self.concurrent:
            self.side.wait_stream(st)
            self.prefix.run(q, k_pool, v_pool, strides, strides, prefix_indices, self.o_p, self.l_p, stream=self.side)
            self.suffix.run(q, k_pool, v_pool, strides, strides, suffix_indices, self.o_s, self.l_s, stream=st)
            st.wait_stream(self.side)
        elif self.suffix_first:
            self.suffix.run(q, k_pool, v_pool, strides, strides, suffix_indices, self.o_s, self.l_s, stream=st)
            self.prefix.run(q, k_pool, v_pool, strides, strides, prefix_indices, self.o_p, self.l_p, stream=st)
        else:
            self.prefix.run(q, k_pool, v_pool, strides, strides, prefix_indices, self.o_p, self.l_p, stream=st)
            self.suffix.run(q, k_pool, v_pool, strides, strides, suffix_indices, self.o_s, self.l_s, stream=st)
        if self.fold_suffix:  # one pass: prefix slots ⊕ suffix state -> o
            self.prefix.contract(o, lse, o_extra=self.o_s, lse_extra=self.l_s, stream=st)
        else:
            self.prefix.contract(self.o_p, self.l_p, stream=st)
            merge_states(self.o_p, self.l_p, self.o_s, self.l_s, o_out=o, lse_out=lse, stream=st)
        return o, lse

    def launches(self) -> int:
        return self.prefix.last_launches() + 1 + self.suffix.last_launches() + (0 if self.fold_suffix else 1)
