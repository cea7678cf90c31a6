"""GPU parity of the tcgen05 kernels against the float64 oracle, and that they are the
kernels actually selected (no silent CUDA-core fallback)."""
import numpy as np
import pytest

import oracle
import synth
from tests.helpers import assert_close, engine_for, run_gpu

pytestmark = pytest.mark.gpu


def _decode_case(cuda_device, *, H_qo=32, H_kv=8, ps=16, dtype="bf16", mask="none", qo=None, kv=None, nc=148,
                 seed=0, layout="NHD", q_scale=1.0):
    kv = np.array(kv if kv is not None else [1, 130, 700, 2049], np.int32)
    qo = np.array(qo if qo is not None else [1] * len(kv), np.int32)
    wl = synth.Workload("tcdec", H_qo, H_kv, 128, ps, dtype, mask, qo, kv)
    inp = synth.make_inputs(wl, device=cuda_device, seed_base=seed, layout=layout, q_scale=q_scale)
    gpu = run_gpu(inp, num_ctas=nc, tile_q=16, kernel="tc")
    assert gpu[2].selected_kernel() == "tc_decode"
    return assert_close(gpu, oracle.attention_from_inputs(inp), dtype, what=f"tc_decode {wl}")


def test_tc_decode_basic(cuda_device):
    _decode_case(cuda_device)


@pytest.mark.parametrize("nc", [1, 7, 148, 296])
def test_tc_decode_num_ctas(cuda_device, nc):
    _decode_case(cuda_device, nc=nc, kv=[5, 1000, 33, 4096, 129, 128])


@pytest.mark.parametrize("H", [(8, 8), (16, 8), (32, 8), (64, 8), (128, 8), (32, 1), (64, 2)])
def test_tc_decode_group_sizes(cuda_device, H):
    _decode_case(cuda_device, H_qo=H[0], H_kv=H[1], nc=64)


@pytest.mark.parametrize("ps", [8, 16, 32, 64, 128, 256])
def test_tc_decode_page_sizes(cuda_device, ps):
    _decode_case(cuda_device, ps=ps, kv=[1, 127, 128, 129, 1000, 2500], nc=32)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("layout", ["NHD", "HND"])
def test_tc_decode_dtypes_layouts(cuda_device, dtype, layout):
    _decode_case(cuda_device, dtype=dtype, layout=layout, nc=20)


@pytest.mark.parametrize("mask", ["causal", "custom"])
def test_tc_decode_multi_token_rows_masks(cuda_device, mask):
    # l_qo up to 4 with g = 4 fills the 16 fused rows (speculative / short append)
    _decode_case(cuda_device, mask=mask, qo=[1, 4, 3, 2, 4], kv=[9, 300, 700, 4, 129], nc=48)


def test_tc_decode_empty_and_zero_requests(cuda_device):
    _decode_case(cuda_device, qo=[1, 1, 0, 1], kv=[0, 17, 5, 0], nc=9)


def test_tc_decode_peaked(cuda_device):
    _decode_case(cuda_device, q_scale=8.0, kv=[300, 2000, 17], qo=[1, 1, 1], nc=30)


def test_tc_decode_c2_full_bench_config(cuda_device):
    """configs[1] at full size in the bench launch configuration (148 CTAs); all 128 requests
    against the oracle (decode is cheap for the oracle)."""
    wl = synth.c2_decode_llama8b()
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = run_gpu(inp, num_ctas=148, tile_q=16, kernel="tc")
    assert gpu[2].selected_kernel() == "tc_decode"
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what="c2 full")


def test_tc_decode_matches_simt(cuda_device):
    """Cross-kernel invariant: tcgen05 and CUDA-core decode agree within tolerance."""
    wl = synth.c2_decode_llama8b(batch=12)
    inp = synth.make_inputs(wl, device=cuda_device)
    a = run_gpu(inp, num_ctas=148, tile_q=16, kernel="tc")
    b = run_gpu(inp, num_ctas=148, tile_q=16, kernel="simt")
    assert np.max(np.abs(a[0] - b[0])) < 1e-2 and np.max(np.abs(a[1] - b[1])) < 1e-3


def test_tc_decode_deterministic(cuda_device):
    wl = synth.c2_decode_llama8b(batch=32)
    inp = synth.make_inputs(wl, device=cuda_device)
    eng = engine_for(wl, num_ctas=148, tile_q=16, kernel="tc")
    a = run_gpu(inp, eng)
    b = run_gpu(inp, eng)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ----------------------------------------------------------- prefill (T_q = 64 / 128 / 256)
def _prefill_case(cuda_device, *, H_qo=64, H_kv=8, ps=16, dtype="bf16", mask="causal", qo=None, kv=None, nc=148,
                  tile_q=128, seed=0, layout="NHD", q_scale=1.0):
    qo = np.array(qo if qo is not None else [70, 129, 1, 300], np.int32)
    kv = np.array(kv if kv is not None else [70, 200, 50, 300], np.int32)
    wl = synth.Workload("tcpre", H_qo, H_kv, 128, ps, dtype, mask, qo, kv)
    inp = synth.make_inputs(wl, device=cuda_device, seed_base=seed, layout=layout, q_scale=q_scale)
    gpu = run_gpu(inp, num_ctas=nc, tile_q=tile_q, kernel="tc")
    assert gpu[2].selected_kernel() == "tc_prefill"
    return assert_close(gpu, oracle.attention_from_inputs(inp), dtype, what=f"tc_prefill {wl} T_q={tile_q}")


@pytest.mark.parametrize("mask", ["none", "causal", "custom"])
@pytest.mark.parametrize("tile_q", [64, 128, 256])
def test_tc_prefill_masks_tiles(cuda_device, mask, tile_q):
    _prefill_case(cuda_device, mask=mask, tile_q=tile_q)


@pytest.mark.parametrize("tile_q", [128, 256])
@pytest.mark.parametrize("nc", [1, 5, 148, 300])
def test_tc_prefill_num_ctas(cuda_device, nc, tile_q):
    _prefill_case(cuda_device, nc=nc, qo=[500, 37, 1000], kv=[700, 37, 1000], tile_q=tile_q)


@pytest.mark.parametrize("tile_q", [128, 256])
@pytest.mark.parametrize("H", [(8, 8), (32, 8), (64, 8), (128, 8), (16, 1)])
def test_tc_prefill_group_sizes(cuda_device, H, tile_q):
    _prefill_case(cuda_device, H_qo=H[0], H_kv=H[1], nc=64, tile_q=tile_q)


@pytest.mark.parametrize("tile_q", [128, 256])
@pytest.mark.parametrize("ps", [8, 32, 128, 256])
def test_tc_prefill_page_sizes(cuda_device, ps, tile_q):
    _prefill_case(cuda_device, ps=ps, nc=40, tile_q=tile_q)


@pytest.mark.parametrize("tile_q", [128, 256])
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("layout", ["NHD", "HND"])
def test_tc_prefill_dtypes_layouts(cuda_device, dtype, layout, tile_q):
    _prefill_case(cuda_device, dtype=dtype, layout=layout, nc=33, tile_q=tile_q)


@pytest.mark.parametrize("tile_q", [128, 256])
def test_tc_prefill_peaked_and_empty(cuda_device, tile_q):
    _prefill_case(cuda_device, q_scale=8.0, qo=[3, 0, 200, 9], kv=[1, 10, 200, 2], mask="causal", nc=17,
                  tile_q=tile_q)


def test_tc_prefill_decode_rows_agree_with_tc_decode(cuda_device):
    """Cross-kernel invariant: l_qo = 1 rows through the prefill kernel (T_q forced to
    128) and the decode kernel (T_q = 16) agree within tolerance."""
    wl = synth.c2_decode_llama8b(batch=16)
    inp = synth.make_inputs(wl, device=cuda_device)
    a = run_gpu(inp, num_ctas=148, tile_q=16, kernel="tc")
    b = run_gpu(inp, num_ctas=148, tile_q=128, kernel="tc")
    assert a[2].selected_kernel() == "tc_decode" and b[2].selected_kernel() == "tc_prefill"
    assert np.max(np.abs(a[0] - b[0])) < 1e-2 and np.max(np.abs(a[1] - b[1])) < 1e-3


def test_tc_prefill_c3_full_bench_config(cuda_device):
    """configs[2] at full size, bench launch configuration (148 CTAs); the shortest, a middle and
    the longest request against the oracle."""
    wl = synth.c3_prefill_llama70b()
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = run_gpu(inp, num_ctas=148, kernel="tc")
    assert gpu[2].selected_kernel() == "tc_prefill"
    order = np.argsort(wl.qo_lens)
    reqs = sorted({int(order[0]), int(order[8]), int(order[-1])})
    from tests.helpers import rows_of_requests
    ref = oracle.attention_from_inputs(inp, req_list=reqs)
    assert_close(gpu, ref, "bf16", rows=rows_of_requests(inp, reqs), what="c3 sampled")


def test_tc_prefill_c3_custom_mask_sampled(cuda_device):
    wl = synth.c3_prefill_llama70b(mask="custom")
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = run_gpu(inp, num_ctas=148, kernel="tc")
    order = np.argsort(wl.qo_lens)
    reqs = sorted({int(order[0]), int(order[5])})
    from tests.helpers import rows_of_requests
    ref = oracle.attention_from_inputs(inp, req_list=reqs)
    assert_close(gpu, ref, "bf16", rows=rows_of_requests(inp, reqs), what="c3 custom sampled")


def test_tc_prefill_deterministic(cuda_device):
    wl = synth.c3_prefill_llama70b(batch=4)
    inp = synth.make_inputs(wl, device=cuda_device)
    eng = engine_for(wl, num_ctas=148, kernel="tc")
    a = run_gpu(inp, eng)
    b = run_gpu(inp, eng)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("tile_q", [16, 128])
def test_tc_pdl_back_to_back_layers(cuda_device, tile_q):
    """BSRA_FLAG_PDL: consecutive independent layers captured in one graph overlap their
    launches; every layer still matches the oracle, including split items (fused contraction
    with the shared workspace across layers)."""
    import torch
    import paper_2501_01005_b200 as bsra
    wl = synth.Workload("pdl", 32, 8, 128, 16, "bf16", "causal" if tile_q == 128 else "none",
                        np.array([1, 1, 1] if tile_q == 16 else [100, 200, 300], np.int32),
                        np.array([5000, 300, 77] if tile_q == 16 else [100, 2000, 300], np.int32))
    layers = [synth.make_inputs(wl, device=cuda_device, seed_base=10 * r) for r in range(4)]
    for inp in layers[1:]:
        inp.kv_page_indices = layers[0].kv_page_indices
    cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", mask=wl.mask, max_batch=3,
                           max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=148, tile_q=tile_q, pdl=True)
    eng = bsra.Engine(cfg, 0)
    i0 = layers[0]
    eng.plan(i0.qo_indptr, i0.kv_page_indptr, i0.kv_last_page_len, i0.sm_scale)
    nq = int(i0.qo_indptr[-1])
    outs = [(torch.empty((nq, 32, 128), device=cuda_device, dtype=torch.bfloat16),
             torch.empty((nq, 32), device=cuda_device)) for _ in layers]
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for inp, (o, l) in zip(layers, outs):
            eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, i0.kv_page_indices, o, l, stream=s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for inp, (o, l) in zip(layers, outs):
        inp.kv_page_indices = i0.kv_page_indices
        assert_close((o.float().cpu().numpy(), l.cpu().numpy()), oracle.attention_from_inputs(inp), "bf16",
                     what="pdl layer")


# ---- cp.async row gather: page sizes a TMA box cannot tile (P:138-139 arbitrary B_c)
def _cp_case(cuda_device, *, ps, layout="NHD", dtype="bf16", mask="none", qo=None, kv=None, nc=37, extra=None):
    """extra: engine_for keywords (cp_async forces the cp.async flavour of the row gather)."""
    kv = np.array(kv if kv is not None else [1, 2, 127, 129, 1000, 2049], np.int32)
    qo = np.array(qo if qo is not None else [1] * len(kv), np.int32)
    wl = synth.Workload("cp", 32, 8, 128, ps, dtype, mask, qo, kv)
    inp = synth.make_inputs(wl, device=cuda_device, layout=layout)
    gpu = run_gpu(inp, num_ctas=nc, tile_q=16, kernel="tc", **(extra or {}))
    assert gpu[2].selected_kernel() == "tc_decode"
    assert_close(gpu, oracle.attention_from_inputs(inp), dtype, what=f"cp gather ps={ps} {layout}")
    return gpu


@pytest.mark.parametrize("cp_async", [False, True], ids=["gather4", "cp_async"])
@pytest.mark.parametrize("ps", [1, 2, 4, 5, 48, 200])
def test_tc_decode_cp_gather_page_sizes(cuda_device, ps, cp_async):
    _cp_case(cuda_device, ps=ps, extra=dict(cp_async=cp_async))


@pytest.mark.parametrize("nc", [1, 148])
def test_tc_decode_cp_gather_split_and_layouts(cuda_device, nc):
    _cp_case(cuda_device, ps=1, layout="HND", dtype="f16", nc=nc, kv=[3000, 5, 700])
    _cp_case(cuda_device, ps=4, mask="causal", qo=[1, 4, 2], kv=[9, 300, 700], nc=nc)


def test_tc_decode_cp_gather_bitwise_equals_tma(cuda_device):
    """BSRA_FLAG_CP_GATHER at B_c = 16 (where TMA boxes apply): same plan, the same values land in
    the same swizzled shared-memory rows, so o and lse are bitwise identical to the TMA gather."""
    import torch
    import paper_2501_01005_b200 as bsra
    wl = synth.Workload("cpb", 32, 8, 128, 16, "bf16", "none", np.ones(5, np.int32),
                        np.array([1, 129, 700, 2049, 4096], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    outs = []
    for cp, ca in ((False, False), (True, False), (True, True)):  # TMA boxes, gather4, cp.async
        cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", max_batch=5, max_total_qo_rows=5,
                               num_ctas=148, tile_q=16, cp_gather=cp, cp_async=ca)
        o, lse, eng = run_gpu(inp, bsra.Engine(cfg, 0))
        outs.append((o, lse))
    for k in (1, 2):
        assert np.array_equal(outs[0][0], outs[k][0]) and np.array_equal(outs[0][1], outs[k][1])
    del torch


def test_c2_page_size_1_full_size_sampled(cuda_device):
    """configs[1] with page size 1 (151,721 one-token pages, the App. B setting P:436) on the
    tensor-core decode kernel; sampled requests."""
    import dataclasses
    from tests.helpers import rows_of_requests
    wl = dataclasses.replace(synth.c2_decode_llama8b(), page_size=1)
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = run_gpu(inp, num_ctas=148, tile_q=16)
    assert gpu[2].selected_kernel() == "tc_decode"
    order = np.argsort(wl.kv_lens)
    reqs = sorted({int(order[0]), int(order[64]), int(order[-1])})
    assert_close(gpu, oracle.attention_from_inputs(inp, req_list=reqs), "bf16", rows=rows_of_requests(inp, reqs),
                 what="c2 ps=1")


# ---- head_dim 64 on the tcgen05 decode kernel (SURVEY §5 AOT set D in {64, 128})
@pytest.mark.parametrize("H,ps,mask,qo", [((32, 8), 16, "none", None), ((16, 2), 8, "causal", [1, 4, 2, 3]),
                                          ((64, 8), 64, "none", None), ((8, 8), 16, "custom", [2, 1, 1, 4])])
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_tc_decode_head_dim_64(cuda_device, H, ps, mask, qo, dtype):
    kv = np.array([1, 130, 700, 2049], np.int32)
    qo = np.array(qo if qo is not None else [1] * 4, np.int32)
    wl = synth.Workload("d64", H[0], H[1], 64, ps, dtype, mask, qo, kv)
    inp = synth.make_inputs(wl, device=cuda_device)
    for nc in (7, 148):
        gpu = run_gpu(inp, num_ctas=nc, tile_q=16, kernel="tc")
        assert gpu[2].selected_kernel() == "tc_decode"
        assert_close(gpu, oracle.attention_from_inputs(inp), dtype, what=f"d64 {H} ps={ps} {mask} nc={nc}")


def test_tc_decode_head_dim_64_matches_simt(cuda_device):
    """Cross-kernel: the same D = 64 decode through the CUDA-core kernel agrees within tolerance."""
    wl = synth.Workload("d64x", 32, 8, 64, 16, "bf16", "none", np.ones(3, np.int32), np.array([33, 700, 5000], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    a = run_gpu(inp, num_ctas=148, tile_q=16, kernel="tc")
    b = run_gpu(inp, num_ctas=148, tile_q=16, kernel="simt")
    assert a[2].selected_kernel() == "tc_decode" and b[2].selected_kernel() == "simt"
    assert np.max(np.abs(a[0] - b[0])) < 1e-2 and np.max(np.abs(a[1] - b[1])) < 1e-3
