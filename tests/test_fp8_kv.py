"""fp8 KV cache — SURVEY §8(f) NEXT-2, the paper's FP8-FP16 mixed-precision attention (P:496-499,
App. F): q and o in fp16/bf16, K/V pools in OCP E4M3 with per-tensor scales (R28).
Every kernel family against the float64 oracle on the same bytes; the tolerance is the q/o
dtype's (the dequantisation is exact, so the error budget of DESIGN.md §9 is unchanged)."""
import ctypes
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import paper_2501_01005_b200 as bsra
import synth
from tests.helpers import assert_close, engine_for, rows_of_requests, run_gpu
from tests.test_ragged_kv import run_ragged


def _fp8(wl):
    return dataclasses.replace(wl, kv_dtype="e4m3")


# ------------------------------------------------------------------ host (no GPU)
def _ws(cfg):
    n = ctypes.c_size_t()
    return bsra.lib().bsra_workspace_bytes(ctypes.byref(cfg), 0, ctypes.byref(n))


def test_fp8_config_validation_host():
    base = dict(H_qo=8, H_kv=2, D=128, page_size=16, max_batch=2, max_total_qo_rows=4, num_ctas=4)
    assert _ws(bsra.make_config(**base, dtype="bf16", kv_dtype="e4m3", k_scale=0.5, v_scale=2.0)) == 0
    assert _ws(bsra.make_config(**base, dtype="f16", kv_dtype="e4m3")) == 0
    assert _ws(bsra.make_config(**base, dtype="bf16", kv_dtype="bf16")) == 0  # == dtype: plain
    assert _ws(bsra.make_config(**base, dtype="f32", kv_dtype="e4m3")) != 0  # q/o stay 16-bit
    assert _ws(bsra.make_config(**base, dtype="bf16", kv_dtype="f16")) != 0
    assert _ws(bsra.make_config(**base, dtype="bf16", kv_dtype="e4m3", k_scale=-1.0)) != 0
    assert _ws(bsra.make_config(**base, dtype="bf16", kv_dtype="e4m3", v_scale=float("inf"))) != 0
    assert "kv_dtype" in bsra.lib().bsra_last_error().decode() or "scale" in bsra.lib().bsra_last_error().decode()


def test_fp8_synth_pools_are_e4m3_bytes_of_scaled_values():
    """The generator stores e4m3(value / scale): dequantised pools keep the bf16 recipe's ranges."""
    wl = _fp8(synth.Workload("g", 8, 2, 64, 4, "bf16", "none", np.array([1, 2], np.int32),
                             np.array([37, 5], np.int32)))
    inp = synth.make_inputs(wl)
    assert inp.k_pool.dtype == torch.float8_e4m3fn and inp.v_pool.element_size() == 1
    v = inp.v_pool.to(torch.float64) * inp.v_scale
    assert float(v.abs().max()) <= 1.0 + 1e-9 and (inp.k_scale, inp.v_scale) == synth.KV_SCALE_E4M3


# ------------------------------------------------------------------ GPU parity
def _case(cuda_device, wl, *, seed=0, layout="NHD", reqs=None, q_scale=1.0, expect=None, **kw):
    inp = synth.make_inputs(wl, device=cuda_device, seed_base=seed, layout=layout, q_scale=q_scale)
    gpu = run_gpu(inp, **kw)
    if expect:
        assert gpu[2].selected_kernel() == expect
    ref = oracle.attention_from_inputs(inp, req_list=reqs)
    rows = rows_of_requests(inp, reqs) if reqs is not None else None
    assert_close(gpu, ref, wl.dtype, rows=rows, what=f"fp8 {wl.name} {kw}")
    return gpu


def _dec(H_qo=32, H_kv=8, ps=16, dtype="bf16", mask="none", qo=None, kv=None):
    kv = np.array(kv if kv is not None else [1, 130, 700, 2049], np.int32)
    qo = np.array(qo if qo is not None else [1] * len(kv), np.int32)
    return _fp8(synth.Workload("f8dec", H_qo, H_kv, 128, ps, dtype, mask, qo, kv))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("layout", ["NHD", "HND"])
def test_fp8_tc_decode_dtypes_layouts(cuda_device, dtype, layout):
    _case(cuda_device, _dec(dtype=dtype), layout=layout, num_ctas=20, tile_q=16, kernel="tc", expect="tc_decode")


@pytest.mark.gpu
@pytest.mark.parametrize("nc", [1, 7, 148, 296])
def test_fp8_tc_decode_num_ctas(cuda_device, nc):
    """Split KV: partial states, the fused in-kernel contraction, v_scale on partials."""
    _case(cuda_device, _dec(kv=[5, 1000, 33, 4096, 129, 128]), num_ctas=nc, tile_q=16, kernel="tc",
          expect="tc_decode")


@pytest.mark.gpu
@pytest.mark.parametrize("ps", [8, 16, 32, 64, 128, 256])
def test_fp8_tc_decode_page_sizes(cuda_device, ps):
    _case(cuda_device, _dec(ps=ps, kv=[1, 127, 128, 129, 1000, 2500]), num_ctas=32, tile_q=16, kernel="tc",
          expect="tc_decode")


@pytest.mark.gpu
@pytest.mark.parametrize("H", [(8, 8), (32, 8), (64, 8), (128, 8), (32, 1)])
def test_fp8_tc_decode_group_sizes(cuda_device, H):
    """Live fused columns kC = 4, 8, 16 (and g > 16 split over q tiles)."""
    _case(cuda_device, _dec(H_qo=H[0], H_kv=H[1]), num_ctas=64, tile_q=16, kernel="tc", expect="tc_decode")


@pytest.mark.gpu
@pytest.mark.parametrize("mask", ["causal", "custom"])
def test_fp8_tc_decode_multi_token_masks(cuda_device, mask):
    _case(cuda_device, _dec(mask=mask, qo=[1, 4, 3, 2, 4], kv=[9, 300, 700, 4, 129]), num_ctas=48, tile_q=16,
          kernel="tc", expect="tc_decode")


@pytest.mark.gpu
def test_fp8_tc_decode_empty_zero_and_peaked(cuda_device):
    _case(cuda_device, _dec(qo=[1, 1, 0, 1], kv=[0, 17, 5, 0]), num_ctas=9, tile_q=16, kernel="tc")
    _case(cuda_device, _dec(kv=[300, 2000, 17], qo=[1, 1, 1]), q_scale=8.0, num_ctas=30, tile_q=16, kernel="tc")


@pytest.mark.gpu
@pytest.mark.parametrize("window,cap", [(33, 0.0), (0, 5.0), (200, 10.0)])
def test_fp8_tc_decode_variants(cuda_device, window, cap):
    """Sliding window (R26) and soft-cap (R27) with the k_scale folded into the logit scale."""
    wl = dataclasses.replace(_dec(mask="causal", qo=[1, 3, 1, 2], kv=[300, 37, 900, 250]), window=window,
                             soft_cap=cap)
    _case(cuda_device, wl, num_ctas=37, tile_q=16, kernel="tc", expect="tc_decode")


@pytest.mark.gpu
def test_fp8_all_codes_including_subnormals(cuda_device):
    """K/V bytes drawn uniformly over all 254 finite E4M3 codes (subnormals, +-0, +-448): the
    converter's exactness on every code, small scales keep the logits sane."""
    wl = _dec(kv=[1, 128, 129, 700])
    inp = synth.make_inputs(wl, device=cuda_device)
    g = torch.Generator(device="cpu").manual_seed(11)
    for pool in (inp.k_pool, inp.v_pool):
        b = torch.randint(0, 254, pool.shape, generator=g, dtype=torch.int32)
        b = torch.where(b >= 0x7F, b + 1, b).to(torch.uint8)  # skip 0x7F (NaN); 0xFF is out of range
        pool.view(torch.uint8).copy_(b.to(cuda_device))
    inp.k_scale, inp.v_scale = 1.0 / 448, 1.0 / 448
    for kernel in ("tc", "simt"):
        gpu = run_gpu(inp, num_ctas=40, tile_q=16, kernel=kernel)
        assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what=f"all codes {kernel}")


@pytest.mark.gpu
def test_fp8_c2_full_size(cuda_device):
    """configs[1] with an E4M3 KV cache at full size in the bench launch configuration (148
    CTAs, the tcgen05 decode kernel); all 128 requests against the oracle."""
    wl = _fp8(synth.c2_decode_llama8b())
    gpu = _case(cuda_device, wl, num_ctas=148, tile_q=16, kernel="tc", expect="tc_decode")
    assert gpu[2].last_launches() == 1


@pytest.mark.gpu
def test_fp8_tc_decode_matches_bf16_pool_of_the_same_values(cuda_device):
    """The converter is exact: the fp8 engine on E4M3 bytes (scale 1) and the bf16 engine on a
    bf16 pool holding the same values give bitwise-identical o and lse."""
    wl = _dec(kv=[5, 1000, 33, 4096, 129, 128])
    inp = synth.make_inputs(wl, device=cuda_device)
    inp.k_scale = inp.v_scale = 1.0
    a = run_gpu(inp, num_ctas=148, tile_q=16, kernel="tc")
    inp16 = dataclasses.replace(inp, wl=dataclasses.replace(wl, kv_dtype=""), k_pool=inp.k_pool.to(torch.bfloat16),
                                v_pool=inp.v_pool.to(torch.bfloat16))
    b = run_gpu(inp16, num_ctas=148, tile_q=16, kernel="tc")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.gpu
def test_fp8_set_kv_scales_between_runs(cuda_device):
    """bsra_set_kv_scales changes the dequantisation of later runs (per-layer scales)."""
    wl = _dec(kv=[100, 900])
    inp = synth.make_inputs(wl, device=cuda_device)
    eng = engine_for(wl, num_ctas=16, tile_q=16, kernel="tc")
    a = run_gpu(inp, eng)
    assert_close(a, oracle.attention_from_inputs(inp), "bf16", what="scales a")
    inp.k_scale, inp.v_scale = 0.05, 0.02
    b = run_gpu(inp, eng)
    assert_close(b, oracle.attention_from_inputs(inp), "bf16", what="scales b")


@pytest.mark.gpu
def test_fp8_ragged_kv(cuda_device):
    """fp8 with the contiguous (ragged) KV layout (NEXT-1): token-coordinate TMA on byte rows."""
    wl = _dec(kv=[1, 130, 700, 2049, 128])
    inp = synth.make_inputs(wl, device=cuda_device)
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=128, dtype=wl.dtype, mask=wl.mask,
                           max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=64, tile_q=16,
                           kernel="tc", ragged_kv=True, kv_dtype="e4m3", k_scale=inp.k_scale, v_scale=inp.v_scale)
    gpu = run_ragged(inp, bsra.Engine(cfg, 0))
    assert gpu[2].selected_kernel() == "tc_decode"
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what="fp8 ragged")


def _pre(mask="causal", ps=16, qo=(70, 129, 1, 300), kv=(70, 200, 50, 300), H=(64, 8), dtype="bf16"):
    return _fp8(synth.Workload("f8pre", H[0], H[1], 128, ps, dtype, mask, np.array(qo, np.int32),
                               np.array(kv, np.int32)))


@pytest.mark.gpu
@pytest.mark.parametrize("mask", ["none", "causal", "custom"])
@pytest.mark.parametrize("tile_q", [64, 128, 256])
def test_fp8_prefill_tc_masks_tiles(cuda_device, mask, tile_q):
    """Prefill tiles with an fp8 KV cache: dequantise-and-gather pass + the tcgen05 prefill kernel
    on the gathered 16-bit copy (f8_gather.cuh); gather + attention (+ contraction) launches."""
    gpu = _case(cuda_device, _pre(mask=mask), num_ctas=148, tile_q=tile_q, expect="tc_prefill")
    assert gpu[2].last_launches() == 3  # gather, attention, contraction (64/128/256-row engines)


@pytest.mark.gpu
@pytest.mark.parametrize("ps", [1, 4, 16, 48, 256])
def test_fp8_prefill_tc_page_sizes(cuda_device, ps):
    """The gather reads any page size (pages smaller than 8 tokens included)."""
    _case(cuda_device, _pre(ps=ps), num_ctas=64, tile_q=128, expect="tc_prefill")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,layout", [("f16", "NHD"), ("bf16", "HND")])
def test_fp8_prefill_tc_dtypes_layouts(cuda_device, dtype, layout):
    _case(cuda_device, _pre(dtype=dtype), layout=layout, num_ctas=37, tile_q=128, expect="tc_prefill")


@pytest.mark.gpu
@pytest.mark.parametrize("nc", [1, 7, 148])
def test_fp8_prefill_tc_split_kv_and_variants(cuda_device, nc):
    """Split KV (partials scaled by v_scale before the contraction), window and soft-cap."""
    wl = dataclasses.replace(_pre(qo=(700, 1, 64), kv=(900, 3000, 64)), window=513, soft_cap=20.0)
    _case(cuda_device, wl, num_ctas=nc, expect="tc_prefill")


@pytest.mark.gpu
def test_fp8_prefill_replan_within_workspace_region(cuda_device):
    """The 16-bit gather copy lives in the caller's workspace, sized by max_total_kv_tokens: plans
    up to the bound reuse it (small -> big -> small), a plan beyond it fails with EBOUNDS and
    keeps the previous plan; the library allocates no device memory (§8(b) ownership)."""
    small, big = _pre(qo=(70, 30), kv=(70, 90)), _pre(qo=(300, 500, 64), kv=(900, 2000, 64))
    eng = engine_for(big, num_ctas=148, tile_q=128, max_batch=4, max_rows=2048)
    assert eng.cfg.max_total_kv_tokens == int(big.kv_lens.sum())
    for wl in (small, big, small):
        inp = synth.make_inputs(wl, device=cuda_device)
        gpu = run_gpu(inp, eng)
        assert gpu[2].selected_kernel() == "tc_prefill"
        assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what=f"replan {wl.kv_lens}")
    too_big = _pre(qo=(300, 500, 64), kv=(900, 2001, 64))
    inp = synth.make_inputs(too_big, device=cuda_device)
    with pytest.raises(bsra.BsraError, match="max_total_kv_tokens"):
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    # a plan without the bound fails loudly instead of allocating
    eng0 = engine_for(small, num_ctas=148, tile_q=128, max_kv=-1)
    inp = synth.make_inputs(small, device=cuda_device)
    with pytest.raises(bsra.BsraError, match="max_total_kv_tokens"):
        eng0.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)


@pytest.mark.gpu
@pytest.mark.parametrize("tile_q", [128, 256])
def test_fp8_prefill_with_pdl(cuda_device, tile_q):
    """BSRA_FLAG_PDL on an fp8 engine with prefill tiles: the prefill kernel reads the copy the
    gather kernel just wrote, so it must not overlap it (launched without PDL); several runs
    back to back on one stream, each checked."""
    wls = [_pre(qo=(700, 1, 64), kv=(900, 3000, 64)), _pre()]
    mx = max(int(w.kv_lens.sum()) for w in wls)
    outs = []
    for wl in wls:
        inp = synth.make_inputs(wl, device=cuda_device)
        cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                               mask=wl.mask, max_batch=4, max_total_qo_rows=2048, num_ctas=148, tile_q=tile_q,
                               kv_dtype="e4m3", k_scale=inp.k_scale, v_scale=inp.v_scale, pdl=True,
                               max_total_kv_tokens=mx)
        eng = bsra.Engine(cfg, 0)
        nq = int(inp.qo_indptr[-1])
        o = torch.full((nq, wl.H_qo, wl.D), float("nan"), device=cuda_device, dtype=torch.bfloat16)
        lse = torch.full((nq, wl.H_qo), float("nan"), device=cuda_device)
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
        outs.append((inp, eng, o, lse))
    for _ in range(3):  # interleaved: each run follows the other engine's kernels on the stream
        for inp, eng, o, lse in outs:
            eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    torch.cuda.synchronize()
    for inp, eng, o, lse in outs:
        assert_close((o.float().cpu().numpy(), lse.cpu().numpy()), oracle.attention_from_inputs(inp), "bf16",
                     what="fp8 prefill + PDL")


@pytest.mark.gpu
def test_fp8_prefill_ragged_kv(cuda_device):
    """fp8 contiguous (ragged) KV with prefill tiles: the gather reads token rows."""
    wl = _pre(qo=(70, 129, 1, 300), kv=(70, 200, 50, 300))
    inp = synth.make_inputs(wl, device=cuda_device)
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=128, dtype=wl.dtype, mask=wl.mask,
                           max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=64, tile_q=128,
                           ragged_kv=True, kv_dtype="e4m3", k_scale=inp.k_scale, v_scale=inp.v_scale,
                           max_total_kv_tokens=int(wl.kv_lens.sum()))
    gpu = run_ragged(inp, bsra.Engine(cfg, 0))
    assert gpu[2].selected_kernel() == "tc_prefill"
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what="fp8 ragged prefill")


@pytest.mark.gpu
def test_fp8_c3_full_size_sampled(cuda_device):
    """configs[2] (ragged causal prefill, 64/8 heads) with an E4M3 KV cache at full size in the
    bench launch configuration; the shortest and one long request checked element by element."""
    wl = _fp8(synth.c3_prefill_llama70b())
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = run_gpu(inp, num_ctas=148)
    assert gpu[2].selected_kernel() == "tc_prefill"
    order = np.argsort(wl.qo_lens)
    reqs = sorted({int(order[0]), int(order[3])})
    assert_close(gpu, oracle.attention_from_inputs(inp, req_list=reqs), "bf16", rows=rows_of_requests(inp, reqs),
                 what="fp8 c3 sampled")


@pytest.mark.gpu
@pytest.mark.parametrize("tile_q", [64, 128])
def test_fp8_prefill_simt_forced(cuda_device, tile_q):
    """kernel="simt": the CUDA-core kernel reads the E4M3 pool directly (no gather)."""
    gpu = _case(cuda_device, _pre(mask="custom"), num_ctas=148, tile_q=tile_q, kernel="simt", expect="simt")
    assert gpu[2].last_launches() == 2


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
def test_fp8_random_small_simt_d64(cuda_device, seed):
    """D = 64 and odd group / page sizes (CUDA-core kernel), ragged masks and empty requests."""
    rng = np.random.default_rng(900 + seed)
    wl = _fp8(synth.random_workload(rng, dtype=["bf16", "f16"][seed % 2], heads=((4, 1), (8, 2), (6, 3)),
                                    page_sizes=(1, 4, 16)))
    _case(cuda_device, wl, seed=seed, num_ctas=int(rng.integers(1, 40)))


@pytest.mark.gpu
@pytest.mark.parametrize("tile_q", [16, 128])
def test_fp8_graph_capture_and_replan(cuda_device, tile_q):
    """run() with an E4M3 cache is graph-capturable (decode kernel; gather pass + prefill): a graph
    captured once replays bitwise-equal to eager runs, also after a re-plan that does not grow the
    gathered 16-bit buffer."""
    import torch
    wl = _dec(qo=[1, 3, 2, 1], kv=[300, 37, 900, 250]) if tile_q == 16 else _pre(qo=(70, 129, 1, 300),
                                                                                  kv=(70, 200, 50, 300))
    inp = synth.make_inputs(wl, device=cuda_device)
    eng = engine_for(wl, num_ctas=64, tile_q=tile_q)
    nq = int(inp.qo_indptr[-1])
    o = torch.zeros((nq, wl.H_qo, wl.D), device=cuda_device, dtype=torch.bfloat16)
    lse = torch.zeros((nq, wl.H_qo), device=cuda_device)
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    eng.set_kv_scales(inp.k_scale, inp.v_scale)
    mbi = None if inp.mask_bit_indptr is None else torch.from_numpy(inp.mask_bit_indptr).to(cuda_device)
    run = lambda: eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse,
                          custom_mask=inp.custom_mask, mask_bit_indptr=mbi)
    run()
    torch.cuda.synchronize()
    eager = (o.clone(), lse.clone())
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        run()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        run()
    o.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(o, eager[0]) and torch.equal(lse, eager[1])
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)  # same lengths
    o.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(o, eager[0]) and torch.equal(lse, eager[1])


@pytest.mark.gpu
@pytest.mark.parametrize("tile_q", [16, 128])
def test_fp8_with_balanced_queues(cuda_device, tile_q):
    """BSRA_FLAG_BALANCE_CTAS with an E4M3 cache: padded plan images drive the fp8 decode kernel
    and the gather + prefill path (re-encoded request table) unchanged."""
    wl = _dec(qo=[1, 1, 1], kv=[5000, 4100, 3000]) if tile_q == 16 else _pre(qo=(300, 129), kv=(3000, 2200))
    inp = synth.make_inputs(wl, device=cuda_device)
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
                           max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=148, tile_q=tile_q,
                           kv_dtype="e4m3", balance_ctas=True, max_total_kv_tokens=int(wl.kv_lens.sum()))
    gpu = run_gpu(inp, bsra.Engine(cfg, 0))
    assert_close(gpu, oracle.attention_from_inputs(inp), wl.dtype, what=f"fp8 balanced T_q={tile_q}")
