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


@pytest.mark.gpu
@pytest.mark.parametrize("pc,sc,conc,fold", [(148, 148, False, True), (64, 84, True, True), (8, 148, False, False),
                                             (8, 140, True, False)])
def test_gpu_composable_fold_paths(cuda_device, pc, sc, conc, fold):
    """bsra_contract with the suffix as extra state (every prefix item split: one launch folds the
    prefix slots and the suffix) and the fallback (prefix rows written through: contraction, then
    merge_states), sequential and on concurrent grids."""
    from tests.helpers import assert_close
    ci = synth.c4_composable(n_branch=16, prefix_len=2048, suffix_len=100, device=cuda_device)
    gpu = _gpu_composable(ci, cuda_device, prefix_ctas=pc, suffix_ctas=sc, concurrent=conc)
    assert gpu[2].fold_suffix == fold
    assert gpu[2].launches() == (3 if fold else 4)
    assert_close(gpu, _oracle(ci, "single"), "bf16", what=f"fold={fold} conc={conc}")


@pytest.mark.gpu
def test_gpu_composable_c4_bench_graph(cuda_device):
    """configs[3] at full size in the bench's launch configuration: prefix on 64 SMs and suffix on
    84 concurrently, captured in a CUDA graph over two layers (two pools) and replayed."""
    import paper_2501_01005_b200 as bsra
    from tests.helpers import assert_close
    cis = [synth.c4_composable(device=cuda_device, seed_base=100 * r) for r in range(2)]
    c0 = cis[0]
    n = c0.q.shape[0]
    comp = bsra.ComposableDecode(H_qo=32, H_kv=8, D=128, page_size=16, n_branch=n, prefix_ctas=64, suffix_ctas=84,
                                 concurrent=True)
    comp.plan(c0.prefix, c0.suffix, c0.sm_scale)
    assert comp.fold_suffix
    # each layer its own page tables (same shapes: the plan is shared)
    idx = [(torch.from_numpy(ci.prefix["kv_page_indices"]).to(cuda_device),
            torch.from_numpy(ci.suffix["kv_page_indices"]).to(cuda_device)) for ci in cis]
    outs = [(torch.full((n, 32, 128), float("nan"), device=cuda_device, dtype=torch.bfloat16),
             torch.full((n, 32), float("nan"), device=cuda_device)) for _ in cis]
    s = torch.cuda.Stream(device=cuda_device)

    def step():
        for ci, (pi, si), (o, l) in zip(cis, idx, outs):
            comp.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, pi, si, o, l, stream=s)
    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    for o, l in outs:
        o.fill_(float("nan"))
        l.fill_(float("nan"))
    with torch.cuda.stream(s):
        g.replay()
        g.replay()
    torch.cuda.synchronize()
    for ci, (o, l) in zip(cis, outs):
        assert_close((o.float().cpu().numpy(), l.cpu().numpy()), _oracle(ci, "single"), "bf16", what="c4 bench graph")


@pytest.mark.gpu
def test_gpu_contract_errors(cuda_device):
    """bsra_contract: EINVAL without BSRA_FLAG_DEFER_CONTRACTION or before a deferred run;
    EUNSUPPORTED for an extra state when rows were written through; decode-only engines cannot
    take the flag."""
    import paper_2501_01005_b200 as bsra
    wl = synth.Workload("ce", 8, 2, 128, 16, "bf16", "none", np.array([4, 4], np.int32), np.array([64, 64], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    with pytest.raises(bsra.BsraError, match="decode-only"):
        bsra.Engine(bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, tile_set=(16,), defer_contraction=True), 0)
    o = torch.empty((8, 8, 128), device=cuda_device, dtype=torch.bfloat16)
    lse = torch.empty((8, 8), device=cuda_device)
    plain = bsra.Engine(bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, max_batch=2, max_total_qo_rows=8,
                                         tile_q=64, num_ctas=2), 0)
    with pytest.raises(bsra.BsraError, match="DEFER"):
        plain.contract(o, lse)
    eng = bsra.Engine(bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, max_batch=2, max_total_qo_rows=8,
                                       tile_q=64, num_ctas=2, defer_contraction=True), 0)
    with pytest.raises(bsra.BsraError, match="no deferred run"):
        eng.contract(o, lse)
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    assert eng.last_launches() == 1
    xo = torch.zeros((8, 8, 128), device=cuda_device)
    xl = torch.full((8, 8), float("-inf"), device=cuda_device)
    with pytest.raises(bsra.BsraError, match="every item split"):  # 2 CTAs, 4 rows: nothing split
        eng.contract(o, lse, o_extra=xo, lse_extra=xl)
    eng.contract(o, lse)  # no extra: nothing to fold, rows written through stay
    torch.cuda.synchronize()
    from tests.helpers import assert_close
    assert_close((o.float().cpu().numpy(), lse.cpu().numpy()), oracle.attention_from_inputs(inp), "bf16",
                 what="deferred, unsplit")


@pytest.mark.gpu
def test_gpu_composable_suffix_first_pdl(cuda_device):
    """Sequential order suffix -> prefix -> bsra_contract with PDL between the launches."""
    from tests.helpers import assert_close
    ci = synth.c4_composable(n_branch=32, prefix_len=4096, suffix_len=200, device=cuda_device)
    gpu = _gpu_composable(ci, cuda_device, prefix_ctas=148, suffix_ctas=148, pdl=True, suffix_first=True)
    assert gpu[2].fold_suffix
    assert_close(gpu, _oracle(ci, "single"), "bf16", what="suffix first, PDL")


@pytest.mark.gpu
def test_gpu_composable_deterministic(cuda_device):
    """The bench's concurrent step (64 + 84 SMs, one bsra_contract) is bitwise reproducible: the
    prefix chunks, the suffix rows and the fold run in a fixed order whatever the timing."""
    ci = synth.c4_composable(n_branch=64, prefix_len=4096, suffix_len=256, device=cuda_device)
    a = _gpu_composable(ci, cuda_device, prefix_ctas=64, suffix_ctas=84, concurrent=True)
    b = _gpu_composable(ci, cuda_device, prefix_ctas=64, suffix_ctas=84, concurrent=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.gpu
def test_gpu_contract_after_replan_needs_a_run(cuda_device):
    """A new plan cancels the pending contraction: bsra_contract between plan() and run() is EINVAL."""
    import paper_2501_01005_b200 as bsra
    wl = synth.Workload("cr", 8, 2, 128, 16, "bf16", "none", np.array([4, 4], np.int32), np.array([640, 64], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    eng = bsra.Engine(bsra.make_config(H_qo=8, H_kv=2, D=128, page_size=16, max_batch=2, max_total_qo_rows=8,
                                       tile_q=64, num_ctas=8, defer_contraction=True), 0)
    o = torch.empty((8, 8, 128), device=cuda_device, dtype=torch.bfloat16)
    lse = torch.empty((8, 8), device=cuda_device)
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    eng.contract(o, lse)
    torch.cuda.synchronize()
    from tests.helpers import assert_close
    assert_close((o.float().cpu().numpy(), lse.cpu().numpy()), oracle.attention_from_inputs(inp), "bf16",
                 what="deferred, split rows")
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    with pytest.raises(bsra.BsraError, match="no deferred run"):
        eng.contract(o, lse)
