"""Composable formats: the shared-prefix + suffix decomposition of a KV
sparse matrix.  CPU: the oracle pins prefix ⊕ suffix ≡ single format.  GPU: the two-engine +
merge_states path (ComposableDecode) against the single-format oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import raw_bits


def _oracle(ci, fmt, **kw):
    f = getattr(ci, fmt)
    return oracle.paged_attention(
        qo_indptr=f["qo_indptr"], kv_page_indptr=f["kv_page_indptr"], kv_last_page_len=f["kv_last_page_len"],
        kv_page_indices=f["kv_page_indices"], q=raw_bits(ci.q), k_pool=raw_bits(ci.k_pool),
        v_pool=raw_bits(ci.v_pool), k_strides=ci.strides, v_strides=ci.strides, H_qo=ci.H_qo, H_kv=ci.H_kv,
        D=ci.D, page_size=ci.page_size, dtype=ci.dtype, sm_scale=ci.sm_scale, **kw)


@pytest.mark.parametrize("suffix_len", [20, 16, 1])
def test_oracle_prefix_oplus_suffix_equals_single(suffix_len):
    ci = synth.c4_composable(n_branch=5, prefix_len=64, suffix_len=suffix_len, H_qo=8, H_kv=2, D=32, page_size=4)
    single = _oracle(ci, "single")
    pre = _oracle(ci, "prefix")
    suf = _oracle(ci, "suffix")
    o, l = oracle.merge(pre[0], pre[1], suf[0], suf[1])
    assert np.max(np.abs(o - single[0])) < 1e-12 and np.max(np.abs(l - single[1])) < 1e-12


def _gpu_composable(ci, dev, **kw):
    import paper_2501_01005_b200 as bsra
    n = ci.q.shape[0]
    comp = bsra.ComposableDecode(H_qo=ci.H_qo, H_kv=ci.H_kv, D=ci.D, page_size=ci.page_size, n_branch=n,
                                 dtype=ci.dtype, **kw)
    comp.plan(ci.prefix, ci.suffix, ci.sm_scale)
    pi = torch.from_numpy(ci.prefix["kv_page_indices"]).to(dev)
    si = torch.from_numpy(ci.suffix["kv_page_indices"]).to(dev)
    o = torch.empty((n, ci.H_qo, ci.D), device=dev, dtype=ci.q.dtype)
    lse = torch.empty((n, ci.H_qo), device=dev)
    comp.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, pi, si, o, lse)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), lse.cpu().numpy(), comp


@pytest.mark.gpu
@pytest.mark.parametrize("n,pre,suf", [(4, 128, 48), (64, 1024, 128), (7, 4096, 1)])
def test_gpu_composable_small(cuda_device, n, pre, suf):
    from tests.helpers import assert_close
    ci = synth.c4_composable(n_branch=n, prefix_len=pre, suffix_len=suf, device=cuda_device)
    gpu = _gpu_composable(ci, cuda_device, prefix_ctas=148, suffix_ctas=148)
    assert gpu[2].prefix.selected_kernel() == "tc_prefill" and gpu[2].suffix.selected_kernel() == "tc_decode"
    ci_cpu = synth.c4_composable(n_branch=n, prefix_len=pre, suffix_len=suf, device="cpu")
    del ci_cpu
    assert_close(gpu, _oracle(ci, "single"), "bf16", what=f"composable n={n}")


@pytest.mark.gpu
def test_gpu_composable_c4_full(cuda_device):
    """configs[3] at full size (8K prefix, 64 x 256 suffixes), bench launch configuration."""
    from tests.helpers import assert_close
    ci = synth.c4_composable(device=cuda_device)
    gpu = _gpu_composable(ci, cuda_device, prefix_ctas=148, suffix_ctas=148)
    assert_close(gpu, _oracle(ci, "single"), "bf16", what="c4 full")
