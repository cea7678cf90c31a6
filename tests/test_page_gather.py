"""Decode page gather layouts (tc_decode): group-major K/V tiles from one 5-D TMA box per page
where the pool strides allow it (page stride a multiple of the head stride, K and V alike), the
half-major 4-D boxes otherwise (padded page strides, K and V in different layouts), and the row
gather (gather4 from four producer warps) for page sizes a box cannot tile — all against the
float64 oracle on the same seeded inputs."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.helpers import assert_close, run_gpu


def _wl(ps, seed=7):
    rng = np.random.default_rng(seed)
    kv = rng.integers(1, 700, size=9).astype(np.int32)
    kv[0] = 1
    kv[1] = 128 * 3  # whole tiles
    return synth.Workload(f"pg{ps}", 32, 8, 128, ps, "bf16", "none", np.ones(9, np.int32), kv)


@pytest.mark.gpu
@pytest.mark.parametrize("ps", [1, 2, 8, 16, 32, 64, 128, 256])
@pytest.mark.parametrize("layout", ["NHD", "HND"])
def test_gpu_decode_page_sizes(cuda_device, ps, layout):
    inp = synth.make_inputs(_wl(ps), device=cuda_device, layout=layout)
    gpu = run_gpu(inp, num_ctas=37, tile_q=16)
    assert gpu[2].selected_kernel() == "tc_decode"
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what=f"ps={ps} {layout}")


@pytest.mark.gpu
@pytest.mark.parametrize("ps", [16, 64])
def test_gpu_decode_padded_page_stride(cuda_device, ps):
    """Page stride = page elements + 64 (not a multiple of the head stride): no 5-D view, the
    half-major boxes take over."""
    inp = synth.make_inputs(_wl(ps, seed=3), device=cuda_device)
    pages = inp.k_pool.shape[0]
    elems = ps * 8 * 128

    def pad(x):
        buf = torch.zeros((pages, elems + 64), device=cuda_device, dtype=x.dtype)
        buf[:, :elems] = x.reshape(pages, elems)
        return buf
    s = (elems + 64, 8 * 128, 128)
    padded = dataclasses.replace(inp, k_pool=pad(inp.k_pool), v_pool=pad(inp.v_pool), k_strides=s, v_strides=s)
    gpu = run_gpu(padded, num_ctas=20, tile_q=16)
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what=f"padded ps={ps}")


@pytest.mark.gpu
def test_gpu_decode_k_nhd_v_hnd(cuda_device):
    """K in NHD and V in HND (different page / head stride ratios): per-tensor 4-D boxes."""
    inp = synth.make_inputs(_wl(16, seed=5), device=cuda_device)
    v_hnd = inp.v_pool.permute(0, 2, 1, 3).contiguous()
    mixed = dataclasses.replace(inp, v_pool=v_hnd, v_strides=(16 * 8 * 128, 128, 16 * 128))
    gpu = run_gpu(mixed, num_ctas=20, tile_q=16)
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what="K NHD / V HND")
