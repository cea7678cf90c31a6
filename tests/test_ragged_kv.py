"""Contiguous (ragged) KV path — SURVEY §8(f) NEXT-1, the layout the paper's App. B compares the
page table against. K/V are [sum l_kv, H_kv, D] tensors indexed by kv_indptr
(bsra_plan_ragged / bsra_run_ragged). The ragged tensors are gathered from the same paged
inputs (synth.ragged_kv), so the float64 oracle on the paged inputs is the reference."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_2501_01005_b200 as bsra
import synth
from tests.helpers import assert_close, rows_of_requests


def ragged_engine(wl, *, num_ctas=148, tile_q=0, kernel="auto", o_dtype=None):
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=128, dtype=wl.dtype, o_dtype=o_dtype,
                           mask=wl.mask, max_batch=max(1, wl.batch), max_total_qo_rows=max(1, int(wl.qo_lens.sum())),
                           num_ctas=num_ctas, tile_q=tile_q, kernel=kernel, ragged_kv=True)
    return bsra.Engine(cfg, 0)


def run_ragged(inp, eng):
    wl = inp.wl
    rk = synth.ragged_kv(inp)
    dev = inp.q.device
    od = bsra.TORCH_DTYPE[eng.cfg.o_dtype]
    nq = int(inp.qo_indptr[-1])
    o = torch.full((nq, wl.H_qo, wl.D), float("nan"), device=dev, dtype=od)
    lse = torch.full((nq, wl.H_qo), float("nan"), device=dev, dtype=torch.float32)
    mbi = None if inp.mask_bit_indptr is None else torch.from_numpy(inp.mask_bit_indptr).to(dev)
    eng.plan_ragged(inp.qo_indptr, rk.kv_indptr, inp.sm_scale)
    eng.run_ragged(inp.q, rk.k, rk.v, rk.k_strides, rk.v_strides, o, lse, custom_mask=inp.custom_mask,
                   mask_bit_indptr=mbi)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), lse.cpu().numpy(), eng


# ------------------------------------------------------------------ host (no GPU)
def test_ragged_kv_gather_matches_page_table():
    """synth.ragged_kv puts token t of request i at row kv_indptr[i] + t (checked element by
    element against the page table, NHD and HND, permuted pages)."""
    wl = synth.Workload("rg", 8, 2, 64, 4, "f32", "none", np.array([1, 2, 1], np.int32),
                        np.array([5, 0, 9], np.int32))
    for layout in ("NHD", "HND"):
        inp = synth.make_inputs(wl, device="cpu", layout=layout, extra_pages=3)
        rk = synth.ragged_kv(inp)
        assert rk.k.shape == (14, 2, 64) and list(rk.kv_indptr) == [0, 5, 5, 14]
        s0, s1, s2 = inp.k_strides
        flat_k, flat_v = inp.k_pool.reshape(-1), inp.v_pool.reshape(-1)
        idx = inp.kv_page_indices.numpy()
        for i in range(wl.batch):
            for t in range(int(wl.kv_lens[i])):
                page = idx[inp.kv_page_indptr[i] + t // wl.page_size]
                for h in range(wl.H_kv):
                    base = page * s0 + (t % wl.page_size) * s1 + h * s2
                    assert torch.equal(rk.k[rk.kv_indptr[i] + t, h], flat_k[base:base + wl.D])
                    assert torch.equal(rk.v[rk.kv_indptr[i] + t, h], flat_v[base:base + wl.D])


def test_ragged_config_rules_host():
    """BSRA_FLAG_RAGGED_KV needs page_size 128 (host-only validation, num_ctas given)."""
    L = bsra.lib()
    n = ctypes.c_size_t()
    ok = bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=128, max_batch=4, max_total_qo_rows=8, num_ctas=4,
                          ragged_kv=True)
    assert L.bsra_workspace_bytes(ctypes.byref(ok), 0, ctypes.byref(n)) == 0 and n.value > 0
    bad = bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, max_batch=4, max_total_qo_rows=8, num_ctas=4,
                           ragged_kv=True)
    assert L.bsra_workspace_bytes(ctypes.byref(bad), 0, ctypes.byref(n)) != 0
    assert b"page_size = 128" in L.bsra_last_error()


# ------------------------------------------------------------------ GPU parity
def _case(cuda_device, wl, *, seed=0, tile_q=0, nc=148, kernel="auto", q_scale=1.0, reqs=None):
    inp = synth.make_inputs(wl, device=cuda_device, seed_base=seed, q_scale=q_scale)
    gpu = run_ragged(inp, ragged_engine(wl, num_ctas=nc, tile_q=tile_q, kernel=kernel))
    ref = oracle.attention_from_inputs(inp, req_list=reqs)
    rows = rows_of_requests(inp, reqs) if reqs is not None else None
    return assert_close(gpu, ref, wl.dtype, rows=rows, what=f"ragged {wl.name} T_q={tile_q} {kernel}"), gpu[2]


@pytest.mark.gpu
@pytest.mark.parametrize("mask", ["none", "causal", "custom"])
@pytest.mark.parametrize("tile_q", [16, 64, 128, 256])
def test_ragged_tc_masks_tiles(cuda_device, mask, tile_q):
    wl = synth.Workload("rg", 32, 8, 128, 16, "bf16", mask, np.array([1, 37, 5, 130, 0, 300], np.int32),
                        np.array([300, 37, 900, 250, 33, 300], np.int32))
    _, eng = _case(cuda_device, wl, tile_q=tile_q, seed=3)
    assert eng.selected_kernel() == ("tc_decode" if tile_q == 16 else "tc_prefill")


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("nc", [1, 7, 148])
def test_ragged_tc_dtypes_ctas(cuda_device, dtype, nc):
    wl = synth.Workload("rg", 64, 8, 128, 16, dtype, "causal", np.array([70, 129, 1, 300], np.int32),
                        np.array([70, 200, 50, 300], np.int32))
    _case(cuda_device, wl, nc=nc)


@pytest.mark.gpu
@pytest.mark.parametrize("wl", [synth.c1_tiny_decode(), synth.Workload("rg64", 8, 2, 64, 16, "bf16", "causal",
                                                                  np.array([3, 40], np.int32),
                                                                  np.array([200, 40], np.int32))],
                         ids=["c1-f32", "d64-bf16"])
def test_ragged_simt(cuda_device, wl):
    _, eng = _case(cuda_device, wl, nc=16)
    assert eng.selected_kernel() == "simt"


@pytest.mark.gpu
def test_ragged_decode_c2_full_sampled(cuda_device):
    """configs[1] at full size through the contiguous path, bench launch configuration."""
    wl = synth.c2_decode_llama8b()
    order = np.argsort(wl.kv_lens)
    _case(cuda_device, wl, tile_q=16, reqs=sorted({int(order[0]), int(order[64]), int(order[-1])}))


@pytest.mark.gpu
def test_ragged_prefill_c3_full_sampled(cuda_device):
    wl = synth.c3_prefill_llama70b()
    order = np.argsort(wl.qo_lens)
    _case(cuda_device, wl, reqs=sorted({int(order[0]), int(order[-1])}))


@pytest.mark.gpu
def test_ragged_and_paged_engines_refuse_the_other_api(cuda_device):
    wl = synth.Workload("rg", 8, 2, 128, 16, "bf16", "none", np.array([1], np.int32), np.array([20], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    eng = ragged_engine(wl)
    with pytest.raises(bsra.BsraError, match="bsra_plan_ragged"):
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len)
    from tests.helpers import engine_for
    pe = engine_for(wl)
    with pytest.raises(bsra.BsraError, match="paged engine"):
        pe.plan_ragged(inp.qo_indptr, np.array([0, 20], np.int32))
