"""The contraction stage: partial states of a split row are merged by ⊕ in the plan's
merge-list order (R17).

CPU: the plan-driven contraction written out with the oracle — every Algorithm-1 item's chunk as
its own float64 partial state, every merge list folded in list order — reproduces the whole
attention; negative controls ("corrupted merge order must fail"): dropping a slot from
a list, or swapping slots between two lists, is caught at the o / lse tolerances, while reversing
a list's order is not an error (⊕ is commutative).
GPU: the fused contraction (inside the decode kernel) and the standalone contraction kernel give
bitwise-identical o and lse for the same plan (the same closed form in the same order)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2501_01005_b200 as bsra
import synth
from oracle import scheduler_ref as S
from synth import raw_bits


def _chunk_state(inp, i, kb, ke):
    """float64 attention state of request i over its keys [kb, ke) (page-aligned chunk)."""
    wl = inp.wl
    ps = wl.page_size
    p0 = int(inp.kv_page_indptr[i])
    n_i = int(inp.kv_page_indptr[i + 1]) - p0
    a, b = kb // ps, -(-ke // ps)
    idx = inp.kv_page_indices.numpy()[p0 + a:p0 + b]
    last = ke - (b - 1) * ps
    q0, q1 = int(inp.qo_indptr[i]), int(inp.qo_indptr[i + 1])
    assert b <= n_i
    return oracle.paged_attention(
        qo_indptr=np.array([0, q1 - q0], np.int32), kv_page_indptr=np.array([0, b - a], np.int32),
        kv_last_page_len=np.array([last], np.int32), kv_page_indices=idx.astype(np.int32),
        q=raw_bits(inp.q)[q0:q1], k_pool=raw_bits(inp.k_pool), v_pool=raw_bits(inp.v_pool), k_strides=inp.k_strides,
        v_strides=inp.v_strides, H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=ps, dtype=wl.dtype,
        sm_scale=inp.sm_scale)


def _contract(inp, plan, lists):
    """Writethrough items + ⊕ over each (possibly corrupted) merge list, in list order."""
    wl = inp.wl
    g = wl.g
    nq = int(inp.qo_indptr[-1])
    o = np.full((nq, wl.H_qo, wl.D), np.nan)
    lse = np.full((nq, wl.H_qo), np.nan)
    part = {}
    for (i, h, t, kb, ke, slot) in plan.items:
        st = _chunk_state(inp, i, kb, ke)
        q0 = int(inp.qo_indptr[i])
        heads = list(range(h * g, (h + 1) * g))
        if slot < 0:
            o[q0:q0 + wl.qo_lens[i], heads] = st[0][:, heads]
            lse[q0:q0 + wl.qo_lens[i], heads] = st[1][:, heads]
        else:  # a partial slot holds only its own (kv head) rows, as on the GPU
            part[slot] = (i, h, (st[0][:, heads], st[1][:, heads]))
    for slots in lists:
        i, h, _ = part[slots[0]]
        heads = list(range(h * g, (h + 1) * g))
        mo, ml = oracle.merge_all([part[s][2] for s in slots])
        q0 = int(inp.qo_indptr[i])
        o[q0:q0 + wl.qo_lens[i], heads] = mo
        lse[q0:q0 + wl.qo_lens[i], heads] = ml
    return o, lse


@pytest.fixture(scope="module")
def split_case():
    wl = synth.Workload("ct", 8, 2, 32, 4, "bf16", "none", np.ones(3, np.int32), np.array([70, 33, 9], np.int32))
    inp = synth.make_inputs(wl)
    plan = S.plan_ref(wl.qo_lens, wl.kv_lens, g=wl.g, H_kv=wl.H_kv, num_ctas=8, tile_set=(16,), align=4)
    assert len(plan.lists) >= 2 and all(len(l[3]) >= 2 for l in plan.lists)
    return inp, plan


def test_plan_driven_contraction_equals_whole(split_case):
    inp, plan = split_case
    ref = oracle.attention_from_inputs(inp)
    o, lse = _contract(inp, plan, [l[3] for l in plan.lists])
    assert np.max(np.abs(o - ref[0])) < 1e-12 and np.max(np.abs(lse - ref[1])) < 1e-12
    # reversed fold order: same state (commutativity), not a corruption
    o2, l2 = _contract(inp, plan, [l[3][::-1] for l in plan.lists])
    assert np.max(np.abs(o2 - ref[0])) < 1e-12 and np.max(np.abs(l2 - ref[1])) < 1e-12


def test_corrupted_merge_lists_are_caught(split_case):
    inp, plan = split_case
    ref = oracle.attention_from_inputs(inp)
    lists = [list(l[3]) for l in plan.lists]
    dropped = [lists[0][1:]] + lists[1:]
    o, lse = _contract(inp, plan, dropped)
    assert np.nanmax(np.abs(lse - ref[1])) > 1e-3  # a missing chunk changes the normaliser
    # swap one slot between two lists of different rows (same chunk count kept)
    a, b = lists[0], lists[1]
    sw = [[b[0]] + a[1:], [a[0]] + b[1:]] + lists[2:]
    try:
        o, lse = _contract(inp, plan, sw)
        err = max(np.nanmax(np.abs(o - ref[0])), np.nanmax(np.abs(lse - ref[1])))
    except (IndexError, ValueError):
        err = np.inf  # shapes of different requests do not even combine
    assert err > 1e-2


@pytest.mark.gpu
def test_fused_and_standalone_contraction_bitwise(cuda_device):
    """Same plan (T_q 16, 148 CTAs) through a decode engine (contraction fused in the kernel) and an
    engine whose tile set allows 64-row tiles (standalone contraction kernel): bitwise equal."""
    wl = synth.Workload("ct", 32, 8, 128, 16, "bf16", "none", np.ones(4, np.int32),
                        np.array([30000, 9000, 17, 4096], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    outs = []
    for tiles in ((16,), (16, 64)):
        cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", max_batch=4, max_total_qo_rows=4,
                               num_ctas=148, tile_set=tiles)  # the heuristic picks T_q = 16 in both
        eng = bsra.Engine(cfg, 0)
        o = torch.empty((4, 32, 128), device=cuda_device, dtype=torch.bfloat16)
        lse = torch.empty((4, 32), device=cuda_device)
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
        eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
        torch.cuda.synchronize()
        outs.append((o, lse, eng.export_plan(), eng.last_launches()))
    assert outs[0][3] == 1 and outs[1][3] == 2  # fused vs separate contraction launch
    assert outs[0][2][3] == 16 and outs[1][2][3] == 16
    assert np.array_equal(outs[0][2], outs[1][2]) and outs[0][2][7] > 0  # same plan, with splits
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
