"""Pins for the Python Algorithm-1 reimplementation (oracle/scheduler_ref.py):
hand traces (tests/golden/alg1_hand_traces.json), the invariants the paper states
(coverage, writethrough iff unsplit, <= 2*#CTA partial tiles, deterministic order),
and the greedy (LPT) balance property. CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import scheduler_ref as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_traces():
    g = json.load(open(os.path.join(GOLDEN, "alg1_hand_traces.json")))
    for c in g["cases"]:
        p = S.plan_ref(c["qo"], c["kv"], g=1, H_kv=1, num_ctas=c["num_ctas"], tile_set=(1,), align=1)
        assert p.T_q == 1 and p.L == c["L"], c["name"]
        spans = sorted((it[3], it[4]) for it in p.items)
        assert spans == sorted(tuple(x) for x in c["chunks"]), c["name"]
        assert p.n_slots == c["n_slots"]
        if c["merge_list"] is None:
            assert p.lists == [] and all(it[5] == -1 for it in p.items)
        else:
            assert p.lists[0][3] == c["merge_list"]
            # merge list order = ascending kv_begin
            begins = {it[5]: it[3] for it in p.items}
            assert [begins[s] for s in p.lists[0][3]] == sorted(begins[s] for s in p.lists[0][3])
        if c["one_chunk_per_cta"]:
            per = [p.cta_indptr[k + 1] - p.cta_indptr[k] for k in range(p.num_ctas)]
            assert max(per) == 1
        if c["num_ctas"] == 1:
            assert p.cta_indptr == [0, 1]


def test_workspace_bound_example():
    w = json.load(open(os.path.join(GOLDEN, "alg1_hand_traces.json")))["workspace_example"]
    assert 2 * w["num_ctas"] * w["T_q"] * w["H_qo"] * (w["D"] + 1) == w["elements"]


@pytest.mark.parametrize("qo,g,expect", [([1] * 128, 4, 16), ([1] * 2, 4, 16), ([5] * 8, 4, 64),
                                         ([64, 2048], 8, 128), ([16] * 4, 1, 16), ([17] * 4, 1, 64)])
def test_select_tile(qo, g, expect):
    """The paper's tile set."""
    assert S.select_tile(qo, g, (16, 64, 128)) == expect


@pytest.mark.parametrize("qo,g,expect", [([64, 2048], 8, 256), ([16] * 4, 8, 128), ([17] * 4, 8, 256),
                                         ([1] * 128, 4, 16), ([4000] * 2, 1, 256)])
def test_select_tile_with_256(qo, g, expect):
    """Extended set with the paired 256-row tile (R20): same rule, one more size."""
    assert S.select_tile(qo, g) == expect


def _check_invariants(p, qo, kv, g, H_kv, mask, num_ctas, T_q):
    # rows and their effective lengths, recomputed here from the definition
    rows = {}
    for i, (lq, lk) in enumerate(zip(qo, kv)):
        fused = lq * g
        for h in range(H_kv):
            for t in range(-(-fused // T_q)):
                if mask == S.MASK_CAUSAL:
                    last_row = min((t + 1) * T_q, fused) - 1
                    e = min(max(lk - lq + last_row // g + 1, 0), lk)
                else:
                    e = lk
                rows[(i, h, t)] = e
    # coverage: chunks of every row partition [0, e)
    by_row = {}
    for it in p.items:
        by_row.setdefault(it[:3], []).append(it)
    assert set(by_row) == set(rows)
    for key, its in by_row.items():
        its = sorted(its, key=lambda x: x[3])
        assert its[0][3] == 0 and its[-1][4] == rows[key]
        for a, b in zip(its, its[1:]):
            assert a[4] == b[3]
        assert all(x[4] - x[3] <= p.L for x in its)
        # DIRECT iff exactly one chunk
        assert (len(its) == 1) == (its[0][5] == -1)
    # <= 2 * #CTA partial tiles (App. D.3)
    assert p.n_slots <= 2 * num_ctas
    # every CTA id valid, queues cover all items
    assert p.cta_indptr[0] == 0 and p.cta_indptr[-1] == len(p.items)
    # greedy balance: max - min CTA cost <= max item cost
    costs = S.cta_costs(p)
    max_item = max((p.T_q + it[4] - it[3] for it in p.items), default=0)
    assert max(costs) - min(costs) <= max_item
    # merge lists in ascending kv_begin
    slot_begin = {it[5]: it[3] for it in p.items if it[5] >= 0}
    for lst in p.lists:
        b = [slot_begin[s] for s in lst[3]]
        assert b == sorted(b)


@pytest.mark.parametrize("seed", range(300))
def test_random_invariants(seed):
    rng = np.random.default_rng(seed)
    B = int(rng.integers(1, 20))
    g = int(rng.choice([1, 2, 4, 8]))
    H_kv = int(rng.choice([1, 2, 8]))
    mask = int(rng.integers(0, 3))
    dist = seed % 3
    if dist == 0:
        kv = rng.integers(0, 3000, B)
    elif dist == 1:
        kv = np.full(B, int(rng.integers(1, 5000)))
    else:  # Zipf-like skew
        kv = np.minimum(rng.zipf(1.5, B) * 37, 200000)
    qo = rng.integers(0, 4, B) if seed % 2 else rng.integers(1, 300, B)
    if mask == S.MASK_CAUSAL:
        kv = np.maximum(kv, qo)
    num_ctas = int(rng.choice([1, 4, 64, 148, 296]))
    align = int(rng.choice([1, 4, 16]))
    p = S.plan_ref(qo, kv, g=g, H_kv=H_kv, mask=mask, num_ctas=num_ctas, align=align)
    _check_invariants(p, [int(x) for x in qo], [int(x) for x in kv], g, H_kv, mask, num_ctas, p.T_q)
    # determinism: identical inputs => identical image
    p2 = S.plan_ref(qo, kv, g=g, H_kv=H_kv, mask=mask, num_ctas=num_ctas, align=align)
    assert np.array_equal(p.image, p2.image)


def test_num_ctas_one_all_direct():
    p = S.plan_ref([1, 3, 7], [100, 2000, 50], g=4, H_kv=2, num_ctas=1, align=16)
    assert all(it[5] == -1 for it in p.items) and p.n_slots == 0


def test_c1_plans_match_survey_table():
    # #CTA=148 -> L=4, 12 chunks all split; #CTA=4 -> L=12, request 0 DIRECT
    p = S.plan_ref([1, 1], [5, 37], g=4, H_kv=1, num_ctas=148, align=4)
    assert p.L == 4 and len(p.items) == 12 and p.n_slots == 12
    p = S.plan_ref([1, 1], [5, 37], g=4, H_kv=1, num_ctas=4, align=4)
    assert p.L == 12 and len(p.items) == 5
    assert sorted((it[3], it[4]) for it in p.items if it[0] == 1) == [(0, 12), (12, 24), (24, 36), (36, 37)]
    assert [it[5] for it in p.items if it[0] == 0] == [-1]


def test_image_header_and_layout():
    p = S.plan_ref([1, 2], [30, 5], g=2, H_kv=2, num_ctas=3, align=4)
    im = p.image
    assert im[0] == S.MAGIC and im[1] == S.VERSION and im[2] == 3 and im[3] == p.T_q and im[4] == p.L
    assert im[5] == len(p.items) and im[6] == len(p.lists) and im[7] == p.n_slots
    expect = S.HEADER_WORDS + 4 + 6 * len(p.items) + len(p.lists) + 1 + p.n_slots + 3 * len(p.lists) + 4 * 2
    assert im.size == expect


@pytest.mark.parametrize("seed", range(200))
def test_window_plan_covers_every_visible_key(seed):
    """Sliding window (R26) in Algorithm 1, checked from the definition: for every fused row of
    every (request, kv head, q tile), the keys it can see (mask AND t >= p - W + 1) lie inside the
    union of the tile's items; each tile's items are disjoint, contiguous, at most L long, start
    on the chunk alignment, and cost the scheduler no more than the windowless plan."""
    rng = np.random.default_rng(9000 + seed)
    B = int(rng.integers(1, 12))
    g = int(rng.choice([1, 4, 8]))
    H_kv = int(rng.choice([1, 2]))
    mask = int(rng.integers(0, 3))
    kv = rng.integers(0, 3000, B)
    qo = rng.integers(0, 3, B) if seed % 2 else rng.integers(1, 200, B)
    if mask == S.MASK_CAUSAL:
        kv = np.maximum(kv, qo)
    W = int(rng.choice([1, 5, 64, 500, 4000]))
    align = int(rng.choice([1, 16, 128]))
    nc = int(rng.choice([1, 8, 148]))
    p = S.plan_ref(qo, kv, g=g, H_kv=H_kv, mask=mask, num_ctas=nc, align=align, window=W)
    by_row = {}
    for it in p.items:
        by_row.setdefault(it[:3], []).append(it)
    for (i, h, t), its in by_row.items():
        its = sorted(its, key=lambda x: x[3])
        for a, b in zip(its, its[1:]):
            assert a[4] == b[3]
        assert its[0][3] % align == 0 and all(x[4] - x[3] <= p.L for x in its)
        lo_cov, hi_cov = its[0][3], its[-1][4]
        lq, lk = int(qo[i]), int(kv[i])
        for f in range(t * p.T_q, min((t + 1) * p.T_q, lq * g)):
            pos = lk - lq + f // g
            vis_lo = max(0, pos - W + 1)
            vis_hi = min(pos + 1, lk) if mask == S.MASK_CAUSAL else lk
            if vis_hi > vis_lo:
                assert lo_cov <= vis_lo and vis_hi <= hi_cov, (i, h, t, f, lo_cov, hi_cov, vis_lo, vis_hi)
    full = S.plan_ref(qo, kv, g=g, H_kv=H_kv, mask=mask, num_ctas=nc, align=align)
    assert sum(x[4] - x[3] for x in p.items) <= sum(x[4] - x[3] for x in full.items)
