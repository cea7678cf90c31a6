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
