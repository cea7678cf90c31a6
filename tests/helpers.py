"""Shared test helpers: run the CUDA path (through the C ABI binding) on synth.Inputs and
compare with the oracle. Imports both sides; neither side imports this."""
import numpy as np
import torch

import oracle
import paper_2501_01005_b200 as bsra
import synth

TOL = {"f32": (1e-5, 1e-5), "f16": (1e-2, 1e-3), "bf16": (1e-2, 1e-3)}  # fp8 KV: q/o dtype's tolerance  # (o, lse): BASELINE north_star


def engine_for(wl, *, num_ctas=0, tile_q=0, tile_set=(16, 64, 128, 256), kernel="auto", o_dtype=None, max_batch=None,
               max_rows=None, max_kv=None, device=0, cp_gather=False, cp_async=False):
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                           o_dtype=o_dtype, mask=wl.mask, max_batch=max_batch or max(1, wl.batch),
                           max_total_qo_rows=max_rows or max(1, int(wl.qo_lens.sum())), num_ctas=num_ctas,
                           tile_set=tile_set, tile_q=tile_q, kernel=kernel, kv_dtype=wl.kv_dtype or None,
                           window=wl.window, soft_cap=wl.soft_cap, alibi=wl.alibi,
                           max_total_kv_tokens=max(0, max_kv) if max_kv is not None else int(wl.kv_lens.astype(np.int64).sum()),
                           cp_gather=cp_gather, cp_async=cp_async, rope_theta=wl.rope_theta,
                           rope_scale=wl.rope_scale)
    return bsra.Engine(cfg, device)


def run_gpu(inp, eng=None, *, o_dtype=None, **kw):
    """plan + run on the inputs' device; returns (o fp32 numpy, lse numpy, engine)."""
    wl = inp.wl
    if eng is None:
        eng = engine_for(wl, o_dtype=o_dtype, **kw)
    dev = inp.q.device
    od = bsra.TORCH_DTYPE[eng.cfg.o_dtype]
    nq = int(inp.qo_indptr[-1])
    o = torch.full((nq, wl.H_qo, wl.D), float("nan"), device=dev, dtype=od)
    lse = torch.full((nq, wl.H_qo), float("nan"), device=dev, dtype=torch.float32)
    mbi = None if inp.mask_bit_indptr is None else torch.from_numpy(inp.mask_bit_indptr).to(dev)
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    if wl.kv_dtype:
        eng.set_kv_scales(inp.k_scale, inp.v_scale)
    eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse,
            custom_mask=inp.custom_mask, mask_bit_indptr=mbi)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), lse.cpu().numpy(), eng


def assert_close(gpu, ref, dtype, rows=None, what=""):
    og, lg = gpu[0], gpu[1]
    orf, lrf = ref
    if rows is not None:
        og, lg, orf, lrf = og[rows], lg[rows], orf[rows], lrf[rows]
    tol_o, tol_l = TOL[dtype]
    assert not np.isnan(og).any(), f"{what}: NaN in o"
    assert not np.isnan(lg).any(), f"{what}: NaN in lse"
    neg_g, neg_r = np.isneginf(lg), np.isneginf(lrf)
    assert np.array_equal(neg_g, neg_r), f"{what}: empty-set rows differ"
    do = float(np.max(np.abs(og - orf), initial=0.0))
    fin = ~neg_r
    dl = float(np.max(np.abs(lg[fin] - lrf[fin]), initial=0.0))
    assert do <= tol_o, f"{what}: max|do| = {do:g} > {tol_o:g}"
    assert dl <= tol_l, f"{what}: max|dlse| = {dl:g} > {tol_l:g}"
    return do, dl


def rows_of_requests(inp, reqs):
    rows = []
    for i in reqs:
        rows.extend(range(int(inp.qo_indptr[i]), int(inp.qo_indptr[i + 1])))
    return np.array(rows, np.int64)
