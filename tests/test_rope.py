"""Fused RoPE (the paper's Query/KeyTransform; R31) on the GPU against
the float64 oracle: the tcgen05 decode kernel's RoPE warps (decode tiles) and the CUDA-core kernel
(other tiles, fp32), at positions up to 128K, with split KV, causal multi-token decode, both
16-bit dtypes, page sizes and layouts, a PDL graph, and configs[1] at full size."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import paper_2501_01005_b200 as bsra
import synth
from tests.helpers import assert_close, rows_of_requests

pytestmark = pytest.mark.gpu


def _rope(wl, theta=10000.0, scale=1.0):
    return dataclasses.replace(wl, rope_theta=theta, rope_scale=scale)


def _run(inp, **kw):
    wl = inp.wl
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                           mask=wl.mask, max_batch=wl.batch, max_total_qo_rows=max(1, int(wl.qo_lens.sum())),
                           rope_theta=wl.rope_theta, rope_scale=wl.rope_scale, **kw)
    eng = bsra.Engine(cfg, 0)
    nq = int(inp.qo_indptr[-1])
    od = bsra.TORCH_DTYPE[cfg.o_dtype]
    o = torch.full((nq, wl.H_qo, wl.D), float("nan"), device=inp.q.device, dtype=od)
    lse = torch.full((nq, wl.H_qo), float("nan"), device=inp.q.device)
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), lse.cpu().numpy(), eng


@pytest.mark.parametrize("theta,scale", [(10000.0, 1.0), (500000.0, 1.0), (10000.0, 4.0)])
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_rope_decode_tc(cuda_device, theta, scale, dtype):
    wl = _rope(synth.Workload("rd", 32, 8, 128, 16, dtype, "none", np.ones(5, np.int32),
                              np.array([1, 17, 300, 2049, 4096], np.int32)), theta, scale)
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = _run(inp, num_ctas=148, tile_q=16)
    assert gpu[2].selected_kernel() == "tc_decode"
    assert_close(gpu, oracle.attention_from_inputs(inp), dtype, what=f"rope decode {theta} {scale}")


@pytest.mark.parametrize("qo,g", [((1, 2, 4), 4), ((1, 1), 16), ((3, 1), 1)])
def test_rope_decode_causal_multi_token(cuda_device, qo, g):
    """Several query tokens per request (live columns 8 / 16): each row at its own position."""
    kv = np.array([70, 130, 1000][:len(qo)], np.int32)
    wl = _rope(synth.Workload("rc", 8 * g if g < 16 else 16, 8 if g < 16 else 1, 128, 16, "bf16", "causal",
                              np.array(qo, np.int32), kv))
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = _run(inp, num_ctas=37, tile_q=16)
    assert gpu[2].selected_kernel() == "tc_decode"
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what=f"rope causal {qo} g={g}")


def test_rope_long_positions_split_kv(cuda_device):
    """128K-token rows split across CTAs (every chunk rotates its keys at their absolute positions,
    then ⊕); exercises the angle reduction at large positions."""
    wl = _rope(synth.Workload("rl", 32, 8, 128, 16, "bf16", "none", np.ones(2, np.int32),
                              np.array([131072, 5000], np.int32)), 500000.0)
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = _run(inp, num_ctas=148, tile_q=16)
    assert gpu[2].export_plan()[7] > 0  # split
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what="rope 128K split")


@pytest.mark.parametrize("ps,layout", [(1, "NHD"), (8, "HND"), (64, "NHD")])
def test_rope_page_sizes_layouts(cuda_device, ps, layout):
    wl = _rope(synth.Workload("rp", 32, 8, 128, ps, "bf16", "none", np.ones(3, np.int32),
                              np.array([33, 700, 129], np.int32)))
    inp = synth.make_inputs(wl, device=cuda_device, layout=layout)
    gpu = _run(inp, num_ctas=64, tile_q=16)
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what=f"rope ps={ps} {layout}")


@pytest.mark.parametrize("tile_q,mask", [(64, "causal"), (128, "causal"), (128, "none")])
def test_rope_prefill_tiles_cuda_core(cuda_device, tile_q, mask):
    """Prefill tiles with RoPE run on the CUDA-core kernel (documented)."""
    wl = _rope(synth.Workload("rq", 32, 8, 128, 16, "bf16", mask, np.array([40, 9, 1], np.int32),
                              np.array([40, 300, 77], np.int32)))
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = _run(inp, num_ctas=64, tile_q=tile_q)
    assert gpu[2].selected_kernel() == "simt"
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what=f"rope prefill T_q={tile_q}")


def test_rope_fp32_tiny(cuda_device):
    """configs[0] shape (fp32, D 64) with RoPE on the CUDA-core kernel, split over 4 CTAs."""
    wl = _rope(synth.c1_tiny_decode())
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = _run(inp, num_ctas=4)
    assert_close(gpu, oracle.attention_from_inputs(inp), "f32", what="rope c1")


def test_rope_rejected_with_fp8_kv():
    cfg = bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, dtype="bf16", kv_dtype="e4m3", rope_theta=1e4,
                           max_batch=1, max_total_qo_rows=1, num_ctas=4)
    with pytest.raises(bsra.BsraError, match="RoPE"):
        bsra.Engine(cfg, 0)


def test_rope_c2_full_size_graph_pdl(cuda_device):
    """configs[1] at full size with RoPE, in the bench's launch configuration (148 CTAs, PDL,
    graph of 2 layers); sampled requests element by element."""
    wl = _rope(synth.c2_decode_llama8b(), 500000.0)
    inps = [synth.make_inputs(wl, device=cuda_device, seed_base=100 * r) for r in range(2)]
    cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", max_batch=128, max_total_qo_rows=128,
                           num_ctas=148, tile_q=16, pdl=True, max_qo_len=1, rope_theta=500000.0)
    eng = bsra.Engine(cfg, 0)
    outs = [(torch.empty((128, 32, 128), device=cuda_device, dtype=torch.bfloat16),
             torch.empty((128, 32), device=cuda_device)) for _ in inps]
    s = torch.cuda.Stream()
    eng.plan(inps[0].qo_indptr, inps[0].kv_page_indptr, inps[0].kv_last_page_len, inps[0].sm_scale)

    def step():
        for inp, (o, l) in zip(inps, outs):
            eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inps[0].kv_page_indices, o, l,
                    stream=s)
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    order = np.argsort(wl.kv_lens)
    reqs = sorted({int(order[0]), int(order[64]), int(order[-1])})
    for r, inp in enumerate(inps):
        inp.kv_page_indices = inps[0].kv_page_indices
        o, l = outs[r]
        assert_close((o.float().cpu().numpy(), l.cpu().numpy()), oracle.attention_from_inputs(inp, req_list=reqs),
                     "bf16", rows=rows_of_requests(inp, reqs), what=f"rope c2 layer {r}")


def test_rope_with_window_softcap_alibi(cuda_device):
    """RoPE (a Query/KeyTransform) composes with the LogitsMask / LogitsTransform variants, which act
    on the rotated logits: sliding window + soft-cap + ALiBi on the decode kernel and the CUDA-core
    kernel (prefill tiles)."""
    base = synth.Workload("rv", 32, 8, 128, 16, "bf16", "causal", np.array([1, 3, 2], np.int32),
                          np.array([900, 300, 2049], np.int32))
    wl = dataclasses.replace(_rope(base), window=256, soft_cap=30.0, alibi=True)
    inp = synth.make_inputs(wl, device=cuda_device)
    ref = oracle.attention_from_inputs(inp)
    for tile_q in (16, 64):
        cfg_kw = dict(num_ctas=37, tile_q=tile_q, window=wl.window, soft_cap=wl.soft_cap, alibi=True)
        gpu = _run(inp, **cfg_kw)
        assert gpu[2].selected_kernel() == ("tc_decode" if tile_q == 16 else "simt")
        assert_close(gpu, ref, "bf16", what=f"rope + variants T_q={tile_q}")


def test_rope_contiguous_kv(cuda_device):
    """RoPE on the contiguous (ragged) KV layout: positions are logical token indices either way."""
    from tests.test_ragged_kv import run_ragged
    wl = _rope(synth.Workload("rr", 32, 8, 128, 16, "bf16", "none", np.ones(3, np.int32),
                              np.array([1, 700, 2049], np.int32)))
    inp = synth.make_inputs(wl, device=cuda_device)
    cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=128, dtype="bf16", max_batch=3, max_total_qo_rows=3,
                           num_ctas=64, tile_q=16, ragged_kv=True, rope_theta=wl.rope_theta)
    gpu = run_ragged(inp, bsra.Engine(cfg, 0))
    assert gpu[2].selected_kernel() == "tc_decode"
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what="rope contiguous KV")
