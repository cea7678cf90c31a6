"""Oracle — TEST INFRASTRUCTURE ONLY.

Plain CPU implementations of what the hot path computes, written from the
paper (arXiv 2501.01005, /root/reference/PAPER.md) and independent of the CUDA
path: the two share no code, and neither imports the other. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.

Contents
  * ``paged_attention``   float64 C oracle (``bsra_oracle.c``), Eq. 1-2 over the BSR page
                          table, causal/custom masks, GQA.
  * ``brute_force``       NumPy: un-page to dense K/V, materialise masked scores, float64
                          softmax. Pins the C oracle (different code, same definition).
  * ``merge`` / ``merge_all``   ⊕ of attention states, float64.
  * ``split_attention``   P contiguous KV shards, each through the oracle, merged in order.
  * ``scheduler_ref``     Algorithm 1 re-implemented in Python.
  * fp8 KV cache          (App. F): K/V stored as OCP E4M3 bytes, q/o in
                          fp16/bf16; element value = scale * E4M3(byte) (R28). Both the
                          C oracle (own decoder) and the brute force (NumPy decoder written from
                          the format definition) take ``kv_dtype="e4m3"``, ``k_scale``, ``v_scale``.

Every function that has no independent pin says so ("parity unpinned") in its
docstring; see DESIGN.md §Oracle.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liborc.so")
_SRC = os.path.join(_HERE, "bsra_oracle.c")
_lib = None

DT_CODE = {"f32": 0, "f16": 1, "bf16": 2, "e4m3": 3}
MASK_CODE = {"none": 0, "causal": 1, "custom": 2}


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2 -fopenmp). Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-o", _SO,
                               _SRC, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        lib.orc_paged_attention.restype = ctypes.c_int
        lib.orc_paged_attention.argtypes = [ctypes.c_int, P, P, P, P, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_double, ctypes.c_double, P, P, P, P, P,
                                            ctypes.c_int, P, P, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                            P, ctypes.c_int, P, P, ctypes.c_int]
        lib.orc_round_dtype.restype = ctypes.c_double
        lib.orc_round_dtype.argtypes = [ctypes.c_double, ctypes.c_int]
        lib.orc_rope_rotate.restype = None
        lib.orc_rope_rotate.argtypes = [P, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        lib.orc_merge.restype = None
        lib.orc_merge.argtypes = [ctypes.c_int64, ctypes.c_int, P, P, P, P, P, P]
        lib.orc_alibi_slope.restype = ctypes.c_double
        lib.orc_alibi_slope.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.orc_decode.restype = ctypes.c_double
        lib.orc_decode.argtypes = [ctypes.c_int, ctypes.c_uint32]
        _lib = lib
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def alibi_slope(h: int, H: int) -> float:
    """ALiBi slope of qo head h of H (C oracle; R30)."""
    return _load().orc_alibi_slope(int(h), int(H))


def alibi_slopes_numpy(H: int) -> np.ndarray:
    """ALiBi slopes written from Press et al.'s construction (different code from the C oracle):
    the geometric sequence 2^(-8/n), 2^(-16/n), ... for n = the largest power of two <= H, then
    every other term of the 2n sequence for the remaining H - n heads."""
    n = 2 ** int(np.floor(np.log2(H)))
    base = 2.0 ** (-8.0 / n)
    pow2 = [base ** (i + 1) for i in range(n)]
    base2 = 2.0 ** (-8.0 / (2 * n))
    extra = [base2 ** (i + 1) for i in range(2 * n)][0::2][:H - n]
    return np.array(pow2 + extra, np.float64)


def decode_scalar(dtype: str, bits: int) -> float:
    return _load().orc_decode(DT_CODE[dtype], int(bits))


def paged_attention(*, qo_indptr, kv_page_indptr, kv_last_page_len, kv_page_indices, q, k_pool, v_pool,
                    k_strides, v_strides, H_qo, H_kv, D, page_size, dtype, mask="none", custom_mask=None,
                    mask_bit_indptr=None, sm_scale, window: int = 0, soft_cap: float = 0.0, alibi: bool = False,
                    kv_dtype: Optional[str] = None, k_scale: float = 1.0, v_scale: float = 1.0,
                    rope_theta: float = 0.0, rope_scale: float = 1.0,
                    req_list: Optional[Sequence[int]] = None, num_threads: int = 0, out=None):
    """float64 oracle (C). Array arguments are host numpy arrays; ``q``/pools hold raw
    element bits (float32, uint16 bits for f16/bf16, uint8 bytes for e4m3 pools).
    ``kv_dtype`` (default: ``dtype``) is the pools' dtype; K/V values are scaled by
    ``k_scale`` / ``v_scale`` (the fp8 KV cache). Returns (o, lse) float64 with
    shapes [sum l_qo, H_qo, D] and [sum l_qo, H_qo]. With ``req_list`` only those requests
    are computed (other rows stay NaN). ``rope_theta`` > 0 applies RoPE to q and k before the
    logits (rotate-half pairs, positions: key t -> t, query row r -> l_kv - l_qo + r; R31)."""
    lib = _load()
    qo_indptr = np.ascontiguousarray(qo_indptr, np.int32)
    kv_page_indptr = np.ascontiguousarray(kv_page_indptr, np.int32)
    kv_last_page_len = np.ascontiguousarray(kv_last_page_len, np.int32)
    kv_page_indices = np.ascontiguousarray(kv_page_indices, np.int32)
    batch = len(qo_indptr) - 1
    nq = int(qo_indptr[-1])
    if out is None:
        o = np.full((nq, H_qo, D), np.nan)
        lse = np.full((nq, H_qo), np.nan)
    else:
        o, lse = out
    ks = np.ascontiguousarray(k_strides, np.int64)
    vs = np.ascontiguousarray(v_strides, np.int64)
    rl = None if req_list is None else np.ascontiguousarray(req_list, np.int32)
    cm = None if custom_mask is None else np.ascontiguousarray(custom_mask, np.uint8)
    mb = None if mask_bit_indptr is None else np.ascontiguousarray(mask_bit_indptr, np.int64)
    q = np.ascontiguousarray(q)
    k_pool = np.asarray(k_pool)
    v_pool = np.asarray(v_pool)
    rc = lib.orc_paged_attention(batch, _ptr(qo_indptr), _ptr(kv_page_indptr), _ptr(kv_last_page_len),
                                 _ptr(kv_page_indices), H_qo, H_kv, D, page_size, DT_CODE[dtype],
                                 DT_CODE[kv_dtype or dtype], float(k_scale), float(v_scale), _ptr(q),
                                 _ptr(k_pool), _ptr(v_pool), _ptr(ks), _ptr(vs), MASK_CODE[mask], _ptr(cm),
                                 _ptr(mb), float(sm_scale), int(window), float(soft_cap), int(bool(alibi)),
                                 float(rope_theta), float(rope_scale), _ptr(rl),
                                 0 if rl is None else len(rl), _ptr(o),
                                 _ptr(lse), int(num_threads))
    if rc != 0:
        raise ValueError(f"orc_paged_attention failed with code {rc}")
    return o, lse


def attention_from_inputs(inp, req_list=None, num_threads=0):
    """Convenience: run the C oracle on a ``synth.Inputs`` (tensors copied to host)."""
    from synth import raw_bits  # input generator only (no method arithmetic)
    wl = inp.wl
    return paged_attention(
        qo_indptr=inp.qo_indptr, kv_page_indptr=inp.kv_page_indptr, kv_last_page_len=inp.kv_last_page_len,
        kv_page_indices=inp.kv_page_indices.cpu().numpy(), q=raw_bits(inp.q), k_pool=raw_bits(inp.k_pool),
        v_pool=raw_bits(inp.v_pool), k_strides=inp.k_strides, v_strides=inp.v_strides, H_qo=wl.H_qo,
        H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
        custom_mask=None if inp.custom_mask is None else inp.custom_mask.cpu().numpy(),
        mask_bit_indptr=inp.mask_bit_indptr, sm_scale=inp.sm_scale, window=wl.window, soft_cap=wl.soft_cap,
        alibi=wl.alibi, kv_dtype=wl.kv_dtype or wl.dtype, k_scale=inp.k_scale, v_scale=inp.v_scale,
        rope_theta=wl.rope_theta, rope_scale=wl.rope_scale, req_list=req_list, num_threads=num_threads)


# ------------------------------------------------------------- brute force ---
def e4m3_to_float64(bits: np.ndarray) -> np.ndarray:
    """OCP FP8 E4M3 bytes -> float64, vectorised from the format definition (R28):
    bias 7; exponent field 0 is subnormal (m/8 * 2^-6); S.1111.111 is NaN; no infinities.
    Independent of the C decoder (table-free, different code)."""
    b = np.asarray(bits, np.uint8).astype(np.int64)
    sign = np.where(b & 0x80, -1.0, 1.0)
    e = (b >> 3) & 0xF
    m = (b & 0x7).astype(np.float64)
    mag = np.where(e == 0, (m / 8.0) * 2.0 ** -6, (1.0 + m / 8.0) * np.exp2(e.astype(np.float64) - 7.0))
    mag = np.where((e == 15) & ((b & 7) == 7), np.nan, mag)
    return sign * mag


def to_float64(bits: np.ndarray, dtype: str) -> np.ndarray:
    """Exact upcast via numpy's own float types (independent of the C decoders)."""
    if dtype == "e4m3":
        return e4m3_to_float64(bits)
    if dtype == "f32":
        return np.asarray(bits, np.float32).astype(np.float64)
    if dtype == "f16":
        return np.asarray(bits, np.uint16).view(np.float16).astype(np.float64)
    u32 = np.asarray(bits, np.uint16).astype(np.uint32) << 16
    return u32.view(np.float32).astype(np.float64)


def brute_force(*, qo_indptr, kv_page_indptr, kv_last_page_len, kv_page_indices, q, k_pool, v_pool,
                k_strides, v_strides, H_qo, H_kv, D, page_size, dtype, mask="none", custom_mask=None,
                mask_bit_indptr=None, sm_scale, window=0, soft_cap=0.0, alibi=False, kv_dtype=None, k_scale=1.0,
                v_scale=1.0, rope_theta=0.0, rope_scale=1.0):
    """NumPy brute force (tiny inputs): dense un-paged K/V per request, the full masked
    score matrix, float64 softmax. Same definition as the C oracle, different code.
    fp8 KV: pools of ``kv_dtype`` scaled by k_scale / v_scale.
    Variants: window W > 0 keeps keys t >= l_kv - l_qo + r - W + 1 (R26);
    soft_cap c > 0 maps the scaled scores through c * tanh(S / c) (R27).
    RoPE (R31), written in complex form (different code from the C oracle's real rotation): the
    pair (x_i, x_{i+D/2}) is the complex number x_i + j x_{i+D/2}, multiplied by e^{j pos theta_i}."""
    qf = to_float64(q, dtype).reshape(-1, H_qo, D)
    kflat = k_scale * to_float64(k_pool, kv_dtype or dtype).reshape(-1)
    vflat = v_scale * to_float64(v_pool, kv_dtype or dtype).reshape(-1)
    g = H_qo // H_kv
    nq = int(qo_indptr[-1])
    o = np.zeros((nq, H_qo, D))
    lse = np.full((nq, H_qo), -np.inf)
    bits = None
    if mask == "custom":
        bits = np.unpackbits(np.asarray(custom_mask, np.uint8), bitorder="little").astype(bool)
    for i in range(len(qo_indptr) - 1):
        q0, q1 = int(qo_indptr[i]), int(qo_indptr[i + 1])
        p0, p1 = int(kv_page_indptr[i]), int(kv_page_indptr[i + 1])
        lq = q1 - q0
        lk = 0 if p1 == p0 else (p1 - p0 - 1) * page_size + int(kv_last_page_len[i])
        if lq == 0:
            continue
        t = np.arange(lk)
        pages = np.asarray(kv_page_indices[p0:p1], np.int64)[t // page_size] if lk else np.zeros(0, np.int64)
        slot = t % page_size
        hk = np.arange(H_kv)
        d = np.arange(D)
        kidx = (pages[:, None, None] * k_strides[0] + slot[:, None, None] * k_strides[1]
                + hk[None, :, None] * k_strides[2] + d[None, None, :])
        vidx = (pages[:, None, None] * v_strides[0] + slot[:, None, None] * v_strides[1]
                + hk[None, :, None] * v_strides[2] + d[None, None, :])
        Kd = kflat[kidx]  # [lk, H_kv, D]
        Vd = vflat[vidx]
        Kr = np.repeat(Kd, g, axis=1)  # GQA: head h uses kv head h // g
        Vr = np.repeat(Vd, g, axis=1)
        Q = qf[q0:q1]
        if rope_theta > 0:  # transformed q / k are tensors of the input dtype (R31)
            Q = round_to_dtype(rope_complex(Q, lk - lq + np.arange(lq), rope_theta, rope_scale), dtype)
            Kr = round_to_dtype(rope_complex(Kr, np.arange(lk), rope_theta, rope_scale), dtype)
        S = sm_scale * np.einsum("rhd,thd->hrt", Q, Kr)  # [H, lq, lk]
        if soft_cap > 0:
            S = soft_cap * np.tanh(S / soft_cap)
        if alibi:  # slope_h * (t - p), p = l_kv - l_qo + r (R30)
            rel = np.arange(lk)[None, :] - (lk - lq + np.arange(lq))[:, None]
            S = S + alibi_slopes_numpy(H_qo)[:, None, None] * rel[None]
        if mask == "none":
            vis = np.ones((lq, lk), bool)
        elif mask == "causal":
            vis = np.arange(lk)[None, :] <= (lk - lq + np.arange(lq))[:, None]
        else:
            b0 = int(mask_bit_indptr[i])
            vis = bits[b0:b0 + lq * lk].reshape(lq, lk)
        if window > 0:
            vis = vis & (np.arange(lk)[None, :] >= (lk - lq + np.arange(lq) - window + 1)[:, None])
        S = np.where(vis[None], S, -np.inf)
        m = S.max(axis=2, initial=-np.inf, keepdims=True)
        msafe = np.where(np.isfinite(m), m, 0.0)
        P = np.where(vis[None], np.exp(S - msafe), 0.0)
        Z = P.sum(axis=2, keepdims=True)
        nz = Z[..., 0] > 0
        l = np.where(nz, (msafe[..., 0] + np.log(np.where(nz, Z[..., 0], 1.0))), -np.inf)
        O = np.einsum("hrt,thd->rhd", P / np.where(Z > 0, Z, 1.0), Vr)
        o[q0:q1] = O
        lse[q0:q1] = l.T
    return o, lse


def rope_complex(x, pos, rope_theta, rope_scale=1.0):
    """RoPE as a complex rotation: x [n, H, D] real with positions pos [n]; z_i = x_i + j x_{i+D/2}
    times e^{j pos theta_i}, theta_i = rope_theta^(-2i/D) / rope_scale (R31)."""
    D = x.shape[-1]
    h = D // 2
    theta = np.power(float(rope_theta), -2.0 * np.arange(h) / D) / rope_scale
    z = x[..., :h] + 1j * x[..., h:]
    z = z * np.exp(1j * np.asarray(pos, np.float64)[:, None, None] * theta[None, None, :])
    return np.concatenate([z.real, z.imag], axis=-1)


def round_to_dtype(x, dtype):
    """Round float64 values to the nearest `dtype` value, ties to even, via numpy's own float
    types (f32, f16) and, for bf16, the f32 bit pattern rounded to its top 16 bits (different code
    from the C oracle's orc_round_dtype). Inputs are O(1): no overflow handling."""
    x = np.asarray(x, np.float64)
    if dtype == "f32":
        return x.astype(np.float32).astype(np.float64)
    if dtype == "f16":
        return x.astype(np.float16).astype(np.float64)
    # bf16: exact in two steps only when the f32 rounding cannot create a tie; use the f64 bits
    b = x.view(np.uint64).astype(np.uint64)
    # keep 1 + 7 fraction bits of the f64 significand (52 - 7 = 45 dropped bits), RN-even
    lsb = (b >> np.uint64(45)) & np.uint64(1)
    b = (b + np.uint64((1 << 44) - 1) + lsb) & ~np.uint64((1 << 45) - 1)
    return b.view(np.float64)


def round_dtype_c(x: float, dtype: str) -> float:
    return _load().orc_round_dtype(float(x), DT_CODE[dtype])


def rope_rotate(x, pos, rope_theta, rope_scale=1.0):
    """The C oracle's RoPE rotation of one vector (float64), for the closed-form pins."""
    x = np.ascontiguousarray(x, np.float64).copy()
    _load().orc_rope_rotate(_ptr(x), x.size, float(pos), float(rope_theta), float(rope_scale))
    return x


def brute_force_from_inputs(inp):
    from synth import raw_bits
    wl = inp.wl
    return brute_force(
        qo_indptr=inp.qo_indptr, kv_page_indptr=inp.kv_page_indptr, kv_last_page_len=inp.kv_last_page_len,
        kv_page_indices=inp.kv_page_indices.cpu().numpy(), q=raw_bits(inp.q), k_pool=raw_bits(inp.k_pool),
        v_pool=raw_bits(inp.v_pool), k_strides=inp.k_strides, v_strides=inp.v_strides, H_qo=wl.H_qo,
        H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
        custom_mask=None if inp.custom_mask is None else inp.custom_mask.cpu().numpy(),
        mask_bit_indptr=inp.mask_bit_indptr, sm_scale=inp.sm_scale, window=wl.window, soft_cap=wl.soft_cap,
        alibi=wl.alibi, kv_dtype=wl.kv_dtype or wl.dtype, k_scale=inp.k_scale, v_scale=inp.v_scale,
        rope_theta=wl.rope_theta, rope_scale=wl.rope_scale)


# --------------------------------------------------------------------- ⊕ ---
def merge(o_a, lse_a, o_b, lse_b):
    """⊕, float64 C implementation, max-shifted; empty state is the
    identity (R3). Shapes: o [..., D], lse [...]."""
    lib = _load()
    o_a = np.ascontiguousarray(o_a, np.float64)
    o_b = np.ascontiguousarray(o_b, np.float64)
    lse_a = np.ascontiguousarray(lse_a, np.float64)
    lse_b = np.ascontiguousarray(lse_b, np.float64)
    D = o_a.shape[-1]
    rows = int(lse_a.size)
    o = np.empty_like(o_a)
    lse = np.empty_like(lse_a)
    lib.orc_merge(rows, D, _ptr(o_a), _ptr(lse_a), _ptr(o_b), _ptr(lse_b), _ptr(o), _ptr(lse))
    return o, lse


def merge_all(states):
    """Left fold of ⊕ in the given order ("composed in any order")."""
    o, lse = states[0]
    for ob, lb in states[1:]:
        o, lse = merge(o, lse, ob, lb)
    return o, lse


def split_attention(inp, P: int, num_threads=0):
    """Sequence split (Ring-Attention/Flash-Decoding use of ⊕): every
    request's pages are cut into P contiguous page ranges (rank r owns pages
    [r*n/P, (r+1)*n/P)); each shard goes through the oracle; states merged in rank order.
    Only meaningful for mask 'none'."""
    from synth import raw_bits
    wl = inp.wl
    assert wl.mask == "none"
    idx = inp.kv_page_indices.cpu().numpy()
    states = []
    for r in range(P):
        indptr = [0]
        sel = []
        last = []
        for i in range(wl.batch):
            p0, p1 = int(inp.kv_page_indptr[i]), int(inp.kv_page_indptr[i + 1])
            n = p1 - p0
            a, b = p0 + (r * n) // P, p0 + ((r + 1) * n) // P
            sel.append(idx[a:b])
            indptr.append(indptr[-1] + (b - a))
            last.append(int(inp.kv_last_page_len[i]) if (b == p1 and b > a) else wl.page_size)
        o, lse = paged_attention(
            qo_indptr=inp.qo_indptr, kv_page_indptr=np.array(indptr, np.int32),
            kv_last_page_len=np.array(last, np.int32), kv_page_indices=np.concatenate(sel).astype(np.int32),
            q=raw_bits(inp.q), k_pool=raw_bits(inp.k_pool), v_pool=raw_bits(inp.v_pool),
            k_strides=inp.k_strides, v_strides=inp.v_strides, H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D,
            page_size=wl.page_size, dtype=wl.dtype, sm_scale=inp.sm_scale, kv_dtype=wl.kv_dtype or wl.dtype,
            k_scale=inp.k_scale, v_scale=inp.v_scale, num_threads=num_threads)
        states.append((o, lse))
    return merge_all(states)
