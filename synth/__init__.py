"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no softmax, no scheduling, no
merge). It only draws lengths and values and lays them out in the paged (BSR)
storage format the paper describes (§3.1.1): a ragged query
tensor indexed by ``qo_indptr`` and a KV pool of pages indexed by
``kv_page_indptr`` / ``kv_page_indices`` / ``kv_last_page_len``.

Recipe:
  * numpy ``Generator(PCG64)`` for lengths, torch generators for values;
    seeds: lengths 0, q 1, k 2, v 3, page permutation 4, custom mask 5
    (each offset by ``seed_base``);
  * q, k ~ N(0, 1); v ~ U(-1, 1) (needed for the 1e-2 o tolerance);
    a "peaked" variant scales q by ``q_scale``;
  * physical page placement is a random permutation of the pool (seed 4), so
    the gather is truly scattered; ``permute=False`` gives contiguous placement;
  * pool layout NHD ``[num_pages, page_size, H_kv, D]`` by default, ``HND``
    (``[num_pages, H_kv, page_size, D]``) available; strides are reported in
    elements as (page, token, head).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

DTYPES = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16, "e4m3": torch.float8_e4m3fn}
# fp8 KV cache: per-tensor scales of the synthetic e4m3 pools. The stored byte is
# the e4m3 rounding of value / scale, so the dequantised values keep the bf16 recipe's ranges
# (k ~ N(0,1), v in [-1, 1]); deliberately not powers of two.
KV_SCALE_E4M3 = (0.03, 0.011)
MASKS = ("none", "causal", "custom")

SEED_LEN, SEED_Q, SEED_K, SEED_V, SEED_PERM, SEED_MASK = 0, 1, 2, 3, 4, 5


@dataclasses.dataclass
class Workload:
    name: str
    H_qo: int
    H_kv: int
    D: int
    page_size: int
    dtype: str
    mask: str
    qo_lens: np.ndarray  # int32 [B]
    kv_lens: np.ndarray  # int32 [B]
    window: int = 0       # sliding window W (0 = off), R26
    soft_cap: float = 0.0  # logits soft-cap c (0 = off), R27
    kv_dtype: str = ""     # "" = dtype; "e4m3" = fp8 KV cache with fp16/bf16 q and o (R28)
    alibi: bool = False    # ALiBi bias (R30)
    rope_theta: float = 0.0  # RoPE base (0 = off), R31
    rope_scale: float = 1.0  # RoPE position interpolation factor

    @property
    def batch(self) -> int:
        return int(len(self.qo_lens))

    @property
    def g(self) -> int:
        return self.H_qo // self.H_kv

    def num_pages(self) -> np.ndarray:
        ps = self.page_size
        return ((self.kv_lens.astype(np.int64) + ps - 1) // ps).astype(np.int64)


# ---------------------------------------------------------------- configs ---
def c1_tiny_decode() -> Workload:
    """BASELINE.json configs[0]: batch 2, 4/1 heads, d 64, page 4, kv {5, 37}, fp32."""
    return Workload("c1_tiny_decode", 4, 1, 64, 4, "f32", "none",
                    np.array([1, 1], np.int32), np.array([5, 37], np.int32))


def sharegpt_like_kv_lens(batch: int = 128, seed: int = SEED_LEN) -> np.ndarray:
    """Log-normal, ShareGPT-like decode lengths clipped to [128, 4096]."""
    r = np.random.default_rng(seed)
    return np.clip(np.round(np.exp(r.normal(np.log(800), 0.9, batch))), 128, 4096).astype(np.int32)


def c2_decode_llama8b(batch: int = 128, seed: int = SEED_LEN) -> Workload:
    """BASELINE.json configs[1]: batched paged decode, 32/8 heads, d 128, page 16, bf16."""
    kv = sharegpt_like_kv_lens(batch, seed)
    return Workload("c2_decode_llama8b", 32, 8, 128, 16, "bf16", "none", np.ones(batch, np.int32), kv)


def c3_prefill_llama70b(batch: int = 16, seed: int = SEED_LEN, mask: str = "causal") -> Workload:
    """BASELINE.json configs[2]: ragged causal prefill, 64/8 heads, d 128, page 16, qo 64..2048."""
    qo = np.random.default_rng(seed).integers(64, 2049, batch).astype(np.int32)
    return Workload("c3_prefill_llama70b", 64, 8, 128, 16, "bf16", mask, qo, qo.copy())


def quest_decode(seq_len: int = 32768, page_budget: int = 512, batch: int = 1, heads: int = 32):
    """Quest fine-grained block-sparse decode (tables eval-sparsity-*): block
    size 16, 32 qo / 32 kv heads, head_dim 128. Quest keeps `page_budget` of each head's
    seq_len/16 pages (query-aware, per head), so every (request, head) is its own BSR row over
    the heads' common pool: a workload of batch*heads single-head "requests" (H_qo = H_kv = 1),
    each with page_budget pages drawn from a pool of batch*heads*seq_len/16 pages (the full
    cache). Returns (workload, extra_pages) for make_inputs(extra_pages=...). Page selection
    itself (Quest's criticality estimate) is out of scope: the kept pages are a seeded random
    subset, which gives the scattered gather the kernel sees."""
    n = batch * heads
    budget = min(page_budget, seq_len // 16)
    wl = Workload(f"quest_{seq_len}_{budget}", 1, 1, 128, 16, "bf16", "none", np.ones(n, np.int32),
                  np.full(n, budget * 16, np.int32))
    return wl, n * (seq_len // 16) - n * budget


def c5_long_decode(batch: int = 4, kv_len: int = 524288) -> Workload:
    """BASELINE.json configs[4]: long-context decode, 32/8 heads, d 128, page 16, kv 512K."""
    return Workload("c5_long_decode", 32, 8, 128, 16, "bf16", "none",
                    np.ones(batch, np.int32), np.full(batch, kv_len, np.int32))


def random_workload(rng: np.random.Generator, *, max_batch=6, max_qo=40, max_kv=90,
                    heads=((4, 1), (4, 4), (8, 1), (8, 2)), dims=(64, 128),
                    page_sizes=(1, 2, 4, 16), dtype="f32", mask=None) -> Workload:
    """Small random workload (ragged, with empty requests) for parity sweeps."""
    B = int(rng.integers(1, max_batch + 1))
    H_qo, H_kv = heads[int(rng.integers(len(heads)))]
    D = int(dims[int(rng.integers(len(dims)))])
    ps = int(page_sizes[int(rng.integers(len(page_sizes)))])
    m = mask or MASKS[int(rng.integers(3))]
    qo = rng.integers(0, max_qo + 1, B).astype(np.int32)
    kv = rng.integers(0, max_kv + 1, B).astype(np.int32)
    if m == "causal":
        kv = np.maximum(kv, qo)  # incremental prefill: l_qo <= l_kv
    return Workload("random", H_qo, H_kv, D, ps, dtype, m, qo, kv)


# ------------------------------------------------------------ materialise ---
@dataclasses.dataclass
class Inputs:
    wl: Workload
    qo_indptr: np.ndarray       # int32 [B+1]
    kv_page_indptr: np.ndarray  # int32 [B+1]
    kv_last_page_len: np.ndarray  # int32 [B]
    kv_page_indices: torch.Tensor  # int32 [nnz]
    q: torch.Tensor             # [sum l_qo, H_qo, D]
    k_pool: torch.Tensor        # NHD [P, ps, H_kv, D] or HND [P, H_kv, ps, D]
    v_pool: torch.Tensor
    k_strides: tuple            # elements (page, token, head)
    v_strides: tuple
    custom_mask: Optional[torch.Tensor]  # uint8 packed bits, LSB first
    mask_bit_indptr: Optional[np.ndarray]  # int64 [B+1]
    sm_scale: float
    k_scale: float = 1.0        # K value = k_scale * stored element (fp8 KV cache, R28)
    v_scale: float = 1.0

    @property
    def device(self):
        return self.q.device


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def page_table(wl: Workload, *, permute=True, seed_base=0, extra_pages=0):
    """Page table in BSR form: kv_page_indptr, kv_page_indices, kv_last_page_len."""
    n = wl.num_pages()
    indptr = np.zeros(wl.batch + 1, np.int64)
    indptr[1:] = np.cumsum(n)
    nnz = int(indptr[-1])
    total_pages = nnz + extra_pages
    if permute:
        perm = np.random.default_rng(SEED_PERM + seed_base).permutation(total_pages)[:nnz]
    else:
        perm = np.arange(nnz)
    last = np.where(n > 0, wl.kv_lens - (n - 1) * wl.page_size, 0).astype(np.int32)
    # requests with pages have last_page_len in [1, page_size]
    return indptr.astype(np.int32), perm.astype(np.int32), last, total_pages


def custom_mask_bits(wl: Workload, *, seed_base=0, density=0.5, causal_and=True):
    """Per request, row-major l_qo x l_kv bits (R9), packed LSB-first.

    Bernoulli(density) AND (optionally) right-aligned lower-triangular, with the
    diagonal t = l_kv - l_qo + r forced visible when it exists."""
    r = np.random.default_rng(SEED_MASK + seed_base)
    bit_indptr = np.zeros(wl.batch + 1, np.int64)
    chunks = []
    for i in range(wl.batch):
        lq, lk = int(wl.qo_lens[i]), int(wl.kv_lens[i])
        bits = r.random((lq, lk)) < density
        if causal_and and lq > 0 and lk > 0:
            rows = np.arange(lq)[:, None]
            cols = np.arange(lk)[None, :]
            lim = lk - lq + rows
            bits &= cols <= lim
            diag_ok = (lim >= 0) & (lim < lk)
            rr = np.nonzero(diag_ok[:, 0])[0]
            bits[rr, (lk - lq + rr)] = True
        chunks.append(bits.reshape(-1))
        bit_indptr[i + 1] = bit_indptr[i] + lq * lk
    flat = np.concatenate(chunks) if chunks else np.zeros(0, bool)
    packed = np.packbits(flat.astype(np.uint8), bitorder="little")
    if packed.size == 0:
        packed = np.zeros(1, np.uint8)
    return packed, bit_indptr


def make_inputs(wl: Workload, *, device="cpu", seed_base=0, permute=True, layout="NHD",
                q_scale=1.0, sm_scale=None, extra_pages=0, mask_bits=None) -> Inputs:
    dt = DTYPES[wl.dtype]
    qo_indptr = np.zeros(wl.batch + 1, np.int32)
    qo_indptr[1:] = np.cumsum(wl.qo_lens)
    kv_indptr, kv_indices, last, total_pages = page_table(wl, permute=permute, seed_base=seed_base,
                                                          extra_pages=extra_pages)
    nq = int(qo_indptr[-1])
    q = torch.randn((nq, wl.H_qo, wl.D), generator=_gen(device, SEED_Q + seed_base), device=device,
                    dtype=torch.float32)
    if q_scale != 1.0:
        q.mul_(q_scale)
    q = q.to(dt)
    if layout == "NHD":
        shape = (total_pages, wl.page_size, wl.H_kv, wl.D)
        strides = (wl.page_size * wl.H_kv * wl.D, wl.H_kv * wl.D, wl.D)
    elif layout == "HND":
        shape = (total_pages, wl.H_kv, wl.page_size, wl.D)
        strides = (wl.page_size * wl.H_kv * wl.D, wl.D, wl.page_size * wl.D)
    else:
        raise ValueError(layout)
    kvt = DTYPES[wl.kv_dtype or wl.dtype]
    ks, vs = KV_SCALE_E4M3 if wl.kv_dtype == "e4m3" else (1.0, 1.0)
    k = torch.empty(shape, device=device, dtype=kvt)
    v = torch.empty(shape, device=device, dtype=kvt)
    # generate in slabs to bound fp32 temporaries on large pools
    slab = max(1, (1 << 26) // max(1, int(np.prod(shape[1:]))))
    gk, gv = _gen(device, SEED_K + seed_base), _gen(device, SEED_V + seed_base)
    for s in range(0, total_pages, slab):
        e = min(total_pages, s + slab)
        kf = torch.randn((e - s,) + shape[1:], generator=gk, device=device)
        vf = torch.rand((e - s,) + shape[1:], generator=gv, device=device) * 2 - 1
        k[s:e] = (kf / ks if ks != 1.0 else kf).to(kvt)
        v[s:e] = (vf / vs if vs != 1.0 else vf).to(kvt)
    cm, mbi = None, None
    if wl.mask == "custom":
        packed, mbi = mask_bits if mask_bits is not None else custom_mask_bits(wl, seed_base=seed_base)
        cm = torch.from_numpy(packed).to(device)
    return Inputs(wl, qo_indptr, kv_indptr, last, torch.from_numpy(kv_indices).to(device), q, k, v,
                  strides, strides, cm, mbi,
                  float(sm_scale) if sm_scale is not None else 1.0 / float(np.sqrt(wl.D)), ks, vs)


def head_slice(inp: Inputs, h0: int, h1: int) -> Inputs:
    """The kv heads [h0, h1) of `inp` and their qo heads [h0*g, h1*g) as a self-contained Inputs
    (data movement only: a contiguous q slice and NHD pools holding only those heads; the page
    table is shared). What one rank of a KV-head-sharded run holds."""
    wl = inp.wl
    g = wl.g
    wl2 = dataclasses.replace(wl, H_qo=(h1 - h0) * g, H_kv=h1 - h0)
    q = inp.q[:, h0 * g:h1 * g].contiguous()

    def cut(pool, st):
        n = pool.numel() // max(1, st[0])
        view = torch.as_strided(pool, (n, wl.page_size, wl.H_kv, wl.D), (st[0], st[1], st[2], 1))
        return view[:, :, h0:h1].contiguous()

    k, v = cut(inp.k_pool, inp.k_strides), cut(inp.v_pool, inp.v_strides)
    st = (wl.page_size * (h1 - h0) * wl.D, (h1 - h0) * wl.D, wl.D)
    return dataclasses.replace(inp, wl=wl2, q=q, k_pool=k, v_pool=v, k_strides=st, v_strides=st)


def request_subset(inp: Inputs, reqs) -> Inputs:
    """Requests `reqs` of `inp` as a self-contained Inputs (data movement only): their q rows, and
    a compact pool holding exactly their pages in BSR order (so a check of a few requests of a
    multi-GB workload copies only those pages to the host). Paged inputs, any layout."""
    wl = inp.wl
    reqs = [int(r) for r in reqs]
    idx = inp.kv_page_indices
    sel = torch.cat([idx[int(inp.kv_page_indptr[i]):int(inp.kv_page_indptr[i + 1])] for i in reqs]).long()
    n = [int(inp.kv_page_indptr[i + 1] - inp.kv_page_indptr[i]) for i in reqs]
    ip = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    qi = np.concatenate([[0], np.cumsum([int(wl.qo_lens[i]) for i in reqs])]).astype(np.int32)
    q = torch.cat([inp.q[int(inp.qo_indptr[i]):int(inp.qo_indptr[i + 1])] for i in reqs])

    def pages(pool, st):
        npg = pool.numel() // max(1, st[0])
        view = torch.as_strided(pool, (npg, st[0]), (st[0], 1))
        return view[sel.to(pool.device)].contiguous().view(-1)

    wl2 = dataclasses.replace(wl, qo_lens=wl.qo_lens[reqs].copy(), kv_lens=wl.kv_lens[reqs].copy())
    cm, mbi = inp.custom_mask, inp.mask_bit_indptr
    if cm is not None:
        raise ValueError("request_subset: custom masks are not re-packed")
    return dataclasses.replace(inp, wl=wl2, qo_indptr=qi, kv_page_indptr=ip,
                               kv_last_page_len=inp.kv_last_page_len[reqs].copy(),
                               kv_page_indices=torch.arange(len(sel), dtype=torch.int32, device=idx.device),
                               q=q, k_pool=pages(inp.k_pool, inp.k_strides), v_pool=pages(inp.v_pool, inp.v_strides))


@dataclasses.dataclass
class RaggedKV:
    """The same keys / values as a paged Inputs, laid out contiguously:
    request i's tokens are rows kv_indptr[i] .. kv_indptr[i+1]-1 of k / v [N, H_kv, D]."""
    kv_indptr: np.ndarray  # int32 [B+1]
    k: torch.Tensor
    v: torch.Tensor
    k_strides: tuple       # elements (token, head)
    v_strides: tuple


def ragged_kv(inp: Inputs) -> RaggedKV:
    """Gathers a paged Inputs' K/V into contiguous ragged tensors (data movement only): token t
    of request i is slot t mod B_c of page indices[kv_page_indptr[i] + t // B_c]."""
    wl = inp.wl
    ps = wl.page_size
    kv_indptr = np.concatenate([[0], np.cumsum(wl.kv_lens.astype(np.int64))]).astype(np.int32)
    idx = inp.kv_page_indices.cpu().numpy().astype(np.int64)
    pages, slots = [], []
    for i in range(wl.batch):
        t = np.arange(int(wl.kv_lens[i]), dtype=np.int64)
        pages.append(idx[inp.kv_page_indptr[i] + t // ps])
        slots.append(t % ps)
    pg = torch.from_numpy(np.concatenate(pages) if pages else np.zeros(0, np.int64)).to(inp.k_pool.device)
    sl = torch.from_numpy(np.concatenate(slots) if slots else np.zeros(0, np.int64)).to(inp.k_pool.device)

    def gather(pool, strides):
        view = torch.as_strided(pool, (pool.numel() // max(1, strides[0]), ps, wl.H_kv, wl.D),
                                (strides[0], strides[1], strides[2], 1))
        return view[pg, sl].contiguous()

    k, v = gather(inp.k_pool, inp.k_strides), gather(inp.v_pool, inp.v_strides)
    st = (wl.H_kv * wl.D, wl.D)
    return RaggedKV(kv_indptr, k, v, st, st)


def raw_bits(t: torch.Tensor) -> np.ndarray:
    """Host numpy view of a tensor's storage: float32 stays float32, 16-bit types as uint16 bits,
    fp8 as uint8 bytes."""
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.float32:
        return t.numpy()
    if t.element_size() == 1:
        return t.view(torch.uint8).numpy()
    return t.view(torch.int16).numpy().view(np.uint16)


# ------------------------------------------------------- composable formats ---
@dataclasses.dataclass
class ComposableInputs:
    """Shared-prefix parallel generation (fig:flashinfer-composable-formats):
    n branches share `prefix_len` tokens of KV; each branch has its own `suffix_len` tokens.
    The same physical pool is described three ways (index arrays only, no data movement):
      single : one BSR, request b = prefix pages + its suffix pages (B_r = 1)
      prefix : one "request" whose l_qo = n query rows (the branches) attend the shared pages
               (the large-B_r block of the paper's figure)
      suffix : n requests over their own suffix pages."""
    q: torch.Tensor          # [n, H_qo, D] one decode query per branch
    k_pool: torch.Tensor
    v_pool: torch.Tensor
    strides: tuple
    single: dict
    prefix: dict
    suffix: dict
    sm_scale: float
    H_qo: int
    H_kv: int
    D: int
    page_size: int
    dtype: str


def c4_composable(n_branch=64, prefix_len=8192, suffix_len=256, H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16",
                  device="cpu", seed_base=0, permute=True) -> ComposableInputs:
    """BASELINE.json configs[3]: 8K shared prefix + 64 branches x 256-token suffixes (decode step).
    Heads follow Llama-3-8B (32/8; an assumption, BASELINE gives only bf16)."""
    ps = page_size
    n_pre = -(-prefix_len // ps)
    n_suf = -(-suffix_len // ps)
    assert prefix_len % ps == 0, "the shared prefix ends on a page boundary (a page is never shared partially)"
    total = n_pre + n_branch * n_suf
    perm = np.random.default_rng(SEED_PERM + seed_base).permutation(total) if permute else np.arange(total)
    pre_pages = perm[:n_pre].astype(np.int32)
    suf_pages = perm[n_pre:].astype(np.int32).reshape(n_branch, n_suf)
    suf_last = suffix_len - (n_suf - 1) * ps
    dt = DTYPES[dtype]
    shape = (total, ps, H_kv, D)
    strides = (ps * H_kv * D, H_kv * D, D)
    q = torch.randn((n_branch, H_qo, D), generator=_gen(device, SEED_Q + seed_base), device=device).to(dt)
    k = torch.empty(shape, device=device, dtype=dt)
    v = torch.empty(shape, device=device, dtype=dt)
    gk, gv = _gen(device, SEED_K + seed_base), _gen(device, SEED_V + seed_base)
    k.copy_(torch.randn(shape, generator=gk, device=device).to(dt))
    v.copy_((torch.rand(shape, generator=gv, device=device) * 2 - 1).to(dt))
    ar = np.arange(n_branch + 1, dtype=np.int32)
    single = dict(qo_indptr=ar.copy(), kv_page_indptr=(ar * (n_pre + n_suf)).astype(np.int32),
                  kv_last_page_len=np.full(n_branch, suf_last, np.int32),
                  kv_page_indices=np.concatenate([np.concatenate([pre_pages, suf_pages[b]])
                                                  for b in range(n_branch)]).astype(np.int32))
    prefix = dict(qo_indptr=np.array([0, n_branch], np.int32), kv_page_indptr=np.array([0, n_pre], np.int32),
                  kv_last_page_len=np.array([ps], np.int32), kv_page_indices=pre_pages.copy())
    suffix = dict(qo_indptr=ar.copy(), kv_page_indptr=(ar * n_suf).astype(np.int32),
                  kv_last_page_len=np.full(n_branch, suf_last, np.int32),
                  kv_page_indices=suf_pages.reshape(-1).copy())
    return ComposableInputs(q, k, v, strides, single, prefix, suffix, 1.0 / float(np.sqrt(D)), H_qo, H_kv, D, ps,
                            dtype)
