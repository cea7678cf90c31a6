"""Attention variants — SURVEY §8(f) NEXT-3, the paper's LogitsMask / LogitsTransform functors
(P:225-228), compiled in (no JIT): sliding window (R26) and logits soft-cap (R27),
on every kernel family, against the float64 oracle on the same inputs."""
import ctypes
import dataclasses

import numpy as np
import pytest

import oracle
import paper_2501_01005_b200 as bsra
import synth
from tests.helpers import assert_close, engine_for, rows_of_requests, run_gpu


def _variant(wl, window=0, soft_cap=0.0, alibi=False):
    return dataclasses.replace(wl, window=window, soft_cap=soft_cap, alibi=alibi)


def _engine(wl, **kw):
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                           mask=wl.mask, max_batch=max(1, wl.batch), max_total_qo_rows=max(1, int(wl.qo_lens.sum())),
                           window=wl.window, soft_cap=wl.soft_cap, alibi=wl.alibi,
                           kv_dtype=wl.kv_dtype or None, max_total_kv_tokens=int(wl.kv_lens.sum()), **kw)
    return bsra.Engine(cfg, 0)


def _case(cuda_device, wl, *, seed=0, reqs=None, q_scale=1.0, **kw):
    inp = synth.make_inputs(wl, device=cuda_device, seed_base=seed, q_scale=q_scale)
    eng = _engine(wl, **kw)
    gpu = run_gpu(inp, eng)
    ref = oracle.attention_from_inputs(inp, req_list=reqs)
    rows = rows_of_requests(inp, reqs) if reqs is not None else None
    assert_close(gpu, ref, wl.dtype, rows=rows, what=f"{wl.name} W={wl.window} cap={wl.soft_cap} {kw}")
    return gpu[2]


# ------------------------------------------------------------------ host
def test_variant_config_validation_host():
    L = bsra.lib()
    n = ctypes.c_size_t()
    for bad in (dict(window=-1), dict(soft_cap=-1.0), dict(soft_cap=float("nan")), dict(soft_cap=float("inf"))):
        cfg = bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, max_batch=2, max_total_qo_rows=4, num_ctas=4, **bad)
        assert L.bsra_workspace_bytes(ctypes.byref(cfg), 0, ctypes.byref(n)) != 0, bad
    ok = bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, max_batch=2, max_total_qo_rows=4, num_ctas=4,
                          window=100, soft_cap=30.0)
    assert L.bsra_workspace_bytes(ctypes.byref(ok), 0, ctypes.byref(n)) == 0


# ------------------------------------------------------------------ GPU parity
_BASE = synth.Workload("var", 32, 8, 128, 16, "bf16", "none", np.array([1, 37, 5, 130, 0, 300], np.int32),
                       np.array([300, 37, 900, 250, 33, 300], np.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("mask", ["none", "causal", "custom"])
@pytest.mark.parametrize("tile_q", [16, 64, 128, 256])
@pytest.mark.parametrize("window,cap", [(1, 0.0), (33, 0.0), (200, 0.0), (0, 5.0), (77, 10.0)])
def test_variants_tc(cuda_device, mask, tile_q, window, cap):
    wl = _variant(dataclasses.replace(_BASE, mask=mask), window, cap)
    eng = _case(cuda_device, wl, seed=3, num_ctas=148, tile_q=tile_q, tile_set=(16, 64, 128, 256))
    assert eng.selected_kernel() == ("tc_decode" if tile_q == 16 else "tc_prefill")


@pytest.mark.gpu
@pytest.mark.parametrize("window,cap", [(5, 0.0), (0, 2.0), (9, 4.0)])
@pytest.mark.parametrize("wl", [synth.c1_tiny_decode(), synth.Workload("d64", 8, 2, 64, 16, "bf16", "causal",
                                                                          np.array([3, 40], np.int32),
                                                                          np.array([200, 40], np.int32))],
                         ids=["c1-f32", "d64-bf16"])
def test_variants_simt(cuda_device, wl, window, cap):
    eng = _case(cuda_device, _variant(wl, window, cap), num_ctas=16)
    assert eng.selected_kernel() == "simt"


@pytest.mark.gpu
@pytest.mark.parametrize("nc", [1, 7, 148])
def test_variants_split_kv(cuda_device, nc):
    """Windows that span many chunks: split items, partial slots and the contraction."""
    wl = _variant(synth.Workload("split", 64, 8, 128, 16, "bf16", "causal", np.array([700, 1, 64], np.int32),
                                 np.array([900, 3000, 64], np.int32)), 513, 20.0)
    _case(cuda_device, wl, num_ctas=nc)


@pytest.mark.gpu
def test_variants_peaked_logits(cuda_device):
    wl = _variant(dataclasses.replace(_BASE, mask="causal"), 50, 3.0)
    _case(cuda_device, wl, q_scale=8.0, num_ctas=148, tile_q=128)


@pytest.mark.gpu
def test_window_decode_c2_full_sampled(cuda_device):
    """configs[1] with a 512-token window: the plan covers only each request's last 512 keys."""
    wl = _variant(synth.c2_decode_llama8b(), 512)
    order = np.argsort(wl.kv_lens)
    reqs = sorted({int(order[0]), int(order[64]), int(order[-1])})
    eng = _case(cuda_device, wl, reqs=reqs, num_ctas=148, tile_q=16)
    im = eng.export_plan()
    n_items = int(im[5])
    base = 16 + int(im[2]) + 1
    kb, ke = im[base + 3 * n_items: base + 4 * n_items], im[base + 4 * n_items: base + 5 * n_items]
    assert int((ke - kb).sum()) <= 8 * (512 + 16) * wl.batch  # window + one page of alignment per row


@pytest.mark.gpu
def test_window_softcap_prefill_c3_full_sampled(cuda_device):
    wl = _variant(synth.c3_prefill_llama70b(), 1024, 30.0)
    order = np.argsort(wl.qo_lens)
    _case(cuda_device, wl, reqs=sorted({int(order[0]), int(order[-1])}), num_ctas=148)


@pytest.mark.gpu
def test_variants_on_contiguous_kv(cuda_device):
    from tests.test_ragged_kv import run_ragged
    wl = _variant(dataclasses.replace(_BASE, mask="causal"), 64, 8.0)
    inp = synth.make_inputs(wl, device=cuda_device, seed_base=5)
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=128, dtype=wl.dtype, mask=wl.mask,
                           max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=148,
                           ragged_kv=True, window=wl.window, soft_cap=wl.soft_cap)
    assert_close(run_ragged(inp, bsra.Engine(cfg, 0)), oracle.attention_from_inputs(inp), "bf16",
                 what="contiguous KV + variants")


# ------------------------------------------------------------------ ALiBi (R30)
def test_alibi_config_validation_host():
    L = bsra.lib()
    n = ctypes.c_size_t()
    cfg = bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, max_batch=2, max_total_qo_rows=4, num_ctas=4, alibi=True)
    assert L.bsra_workspace_bytes(ctypes.byref(cfg), 0, ctypes.byref(n)) == 0
    cfg.alibi = 2
    assert L.bsra_workspace_bytes(ctypes.byref(cfg), 0, ctypes.byref(n)) != 0


@pytest.mark.gpu
@pytest.mark.parametrize("mask", ["none", "causal", "custom"])
@pytest.mark.parametrize("tile_q", [16, 64, 128, 256])
@pytest.mark.parametrize("window,cap", [(0, 0.0), (200, 0.0), (0, 10.0)])
def test_alibi_tc(cuda_device, mask, tile_q, window, cap):
    wl = _variant(dataclasses.replace(_BASE, mask=mask), window, cap, alibi=True)
    eng = _case(cuda_device, wl, seed=5, num_ctas=148, tile_q=tile_q, tile_set=(16, 64, 128, 256))
    assert eng.selected_kernel() == ("tc_decode" if tile_q == 16 else "tc_prefill")


@pytest.mark.gpu
@pytest.mark.parametrize("H", [(32, 8), (40, 8), (12, 4)])
def test_alibi_head_counts(cuda_device, H):
    """Non-power-of-two head counts use the interleaved extra slopes (Press et al.)."""
    wl = _variant(synth.Workload("alibiH", H[0], H[1], 128, 16, "bf16", "causal", np.array([1, 9, 130], np.int32),
                                 np.array([700, 9, 400], np.int32)), alibi=True)
    _case(cuda_device, wl, num_ctas=64)


@pytest.mark.gpu
@pytest.mark.parametrize("wl", [synth.c1_tiny_decode(), synth.Workload("d64", 8, 2, 64, 16, "bf16", "causal",
                                                                          np.array([3, 40], np.int32),
                                                                          np.array([200, 40], np.int32))],
                         ids=["c1-f32", "d64-bf16"])
def test_alibi_simt(cuda_device, wl):
    eng = _case(cuda_device, _variant(wl, alibi=True), num_ctas=16)
    assert eng.selected_kernel() == "simt"


@pytest.mark.gpu
@pytest.mark.parametrize("tile_q", [16, 128])
def test_alibi_fp8_kv(cuda_device, tile_q):
    """ALiBi with an E4M3 KV cache: fp8 decode kernel and the gather + prefill path."""
    wl = dataclasses.replace(_variant(dataclasses.replace(_BASE, mask="causal"), alibi=True), kv_dtype="e4m3")
    _case(cuda_device, wl, num_ctas=148, tile_q=tile_q, tile_set=(16, 64, 128, 256))


@pytest.mark.gpu
def test_alibi_split_kv(cuda_device):
    wl = _variant(synth.Workload("split", 64, 8, 128, 16, "bf16", "causal", np.array([700, 1, 64], np.int32),
                                 np.array([900, 3000, 64], np.int32)), 0, 0.0, alibi=True)
    for nc in (1, 7, 148):
        _case(cuda_device, wl, num_ctas=nc)
