"""Pins for Algorithm 1's ORDERING steps (alg:load-balancing lines 5-11):
descending sort by chunk length with ties on ascending work index, and the min-heap greedy
with ties on the lowest CTA id (R15). Each case in
tests/golden/alg1_order_traces.json was worked by hand and lists the exact per-CTA queues,
so a plan that only satisfies the order-free invariants (coverage, LPT balance) fails here.

Negative controls: the two plausible misreadings the round-1 review found passing every
other pin — sorting ascending, and breaking CTA-cost ties toward the highest id — plus a
descending-work-index tie-break are injected into oracle/scheduler_ref.plan_ref and must
make the goldens fail. The C++ scheduler (bsra_plan_host) is checked against the same
goldens directly. CPU only."""
import heapq as _heapq
import json
import os

import numpy as np
import pytest

from oracle import scheduler_ref as S

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "alg1_order_traces.json")))
CASES = GOLDEN["cases"]


def _work_ids(case):
    """(request, kv_begin) of every work index w, from the golden's chunk list in (row, j) order."""
    req, out = -1, []
    for b, _e in case["chunks"]:
        if b == 0:
            req += 1
        out.append((req, b))
    return {k: w for w, k in enumerate(out)}


def _queues_from_items(case, items, cta_indptr):
    wid = _work_ids(case)
    return [[wid[(it[0], it[3])] for it in items[cta_indptr[c]:cta_indptr[c + 1]]]
            for c in range(case["num_ctas"])]


def _plan(case):
    return S.plan_ref(case["qo"], case["kv"], g=1, H_kv=1, num_ctas=case["num_ctas"], tile_set=(1,),
                      align=case["align"])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_order_trace(case):
    p = _plan(case)
    assert p.T_q == 1 and p.L == case["L"]
    wid = _work_ids(case)
    # chunks and slots per work index
    got = {}
    for it in p.items:
        got[wid[(it[0], it[3])]] = (it[3], it[4], it[5])
    assert [list(got[w][:2]) for w in range(len(case["chunks"]))] == case["chunks"]
    assert [got[w][2] for w in range(len(case["chunks"]))] == case["slots"]
    assert [lst[3] for lst in p.lists] == case.get("merge_lists", [])
    assert _queues_from_items(case, p.items, p.cta_indptr) == case["queues"]
    assert S.cta_costs(p) == case["cta_costs"]


class _HighIdHeap:
    """heapq shim whose pops break cost ties toward the HIGHEST CTA id (a misreading)."""

    @staticmethod
    def heapify(h):
        h[:] = [(c, -k) for c, k in h]
        _heapq.heapify(h)

    @staticmethod
    def heappop(h):
        c, k = _heapq.heappop(h)
        return c, -k

    @staticmethod
    def heappush(h, x):
        _heapq.heappush(h, (x[0], -x[1]))


def _mutated_sort(chunk_key):
    """A `sorted` that re-keys plan_ref's chunk sort (5-tuples (w, row, j, begin, end)) and
    leaves every other call alone."""
    import builtins

    def _sorted(seq, key=None, reverse=False):
        seq = list(seq)
        if key is not None and seq and isinstance(seq[0], tuple) and len(seq[0]) == 5:
            return builtins.sorted(seq, key=chunk_key)
        return builtins.sorted(seq, key=key, reverse=reverse)
    return _sorted


_asc = _mutated_sort(lambda c: (c[4] - c[3], c[0]))
_desc_w_sorted = _mutated_sort(lambda c: (-(c[4] - c[3]), -c[0]))


MUTATIONS = {
    "ascending sort": ("sorted", _asc),
    "highest CTA id on ties": ("heapq", _HighIdHeap),
    "descending work index on equal lengths": ("sorted", _desc_w_sorted),
}


@pytest.mark.parametrize("mutation", sorted(MUTATIONS))
def test_mutations_fail_the_goldens(monkeypatch, mutation):
    """Negative control: each misreading changes at least one golden's queues — and exactly to
    the hand-worked alternative where the golden records one."""
    attr, repl = MUTATIONS[mutation]
    monkeypatch.setattr(S, attr, repl, raising=False)
    differs = 0
    for case in CASES:
        p = _plan(case)
        q = _queues_from_items(case, p.items, p.cta_indptr)
        if q != case["queues"]:
            differs += 1
        alt = case.get("mutations_differ", {}).get(mutation)
        if alt is not None:
            assert q == alt, (case["name"], mutation, q)
    assert differs >= 1, f"mutation '{mutation}' passes every ordering golden"


def test_cpp_scheduler_matches_order_goldens():
    """The C++ scheduler (bsra_plan_host) against the same hand traces, not only against plan_ref."""
    bsra = pytest.importorskip("paper_2501_01005_b200")
    for case in CASES:
        qo, kv = np.array(case["qo"]), np.array(case["kv"])
        # page size 1 => BSR pages are tokens, last_page_len 1
        qi = np.concatenate([[0], np.cumsum(qo)]).astype(np.int32)
        ki = np.concatenate([[0], np.cumsum(kv)]).astype(np.int32)
        last = np.ones(len(kv), np.int32)
        cfg = bsra.make_config(H_qo=1, H_kv=1, D=128, page_size=1, dtype="bf16", max_batch=len(qo),
                               max_total_qo_rows=int(qo.sum()), num_ctas=case["num_ctas"], tile_set=(16,),
                               kv_chunk_align=case["align"])
        im = bsra.plan_host(cfg, case["num_ctas"], qi, ki, last)
        nc, n_items = int(im[2]), int(im[5])
        assert int(im[4]) == case["L"], case["name"]
        ind = im[S.HEADER_WORDS:S.HEADER_WORDS + nc + 1]
        base = S.HEADER_WORDS + nc + 1
        req = im[base:base + n_items]
        kb = im[base + 3 * n_items:base + 4 * n_items]
        items = [(int(req[j]), 0, 0, int(kb[j])) for j in range(n_items)]
        assert _queues_from_items(case, items, [int(x) for x in ind]) == case["queues"], case["name"]
