"""Algorithm 1 (§3.3.1, alg:load-balancing) — Python reimplementation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). The C++ host scheduler in
paper_2501_01005_b200/csrc must emit a byte-identical plan image; nothing here
is shared with it. Exact integer arithmetic only.

Paper steps and the readings that make them deterministic (R11-R20):
  1. T_q = minimal tile >= average head-fused query length (§3.2.2, PAPER.md:205;
     App. A): T_q = min{T in T_set : T*B >= sum_i l_qo(i)*g}, else max(T_set).
  2. rows = (request, kv head, q-tile) (R12: "head dimension is omitted for simplicity");
     each row charges its causal-effective KV length e (R13).
  3. L_kv = ceil(sum e / #CTA), floored at L_min and 1, rounded UP to
     the alignment (default page size, R11).
  4. split each row into chunks of at most L_kv, fixed stride from 0 (R14);
     work index w in (row, j) order; a row with e = 0 still gets one empty chunk.
  5. sort by descending length, ties by ascending w (R15).
  6. min-heap of (cost, cta); pop min, assign, push cost + alpha*T_q + beta*len
     (cost(l_q, l_kv) = alpha*l_q + beta*l_kv; R16).
  7. unsplit rows write through (slot -1, App. D.2); split rows get
     consecutive partial slots in chunk order and one merge list each (R17).
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

MAGIC = 0x41525342  # 'BSRA' little-endian
VERSION = 1
HEADER_WORDS = 16
MASK_NONE, MASK_CAUSAL, MASK_CUSTOM = 0, 1, 2


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def select_tile(qo_lens, g, tile_set=(16, 64, 128, 256)) -> int:
    """§3.2.2 heuristic, integer form: smallest T with T*B >= sum(l_qo*g)."""
    B = len(qo_lens)
    S = int(sum(int(x) for x in qo_lens)) * g
    for T in sorted(tile_set):
        if T * B >= S:
            return T
    return max(tile_set)


@dataclass
class Plan:
    num_ctas: int
    T_q: int
    L: int
    items: list  # queue order: (req, kvh, qtile, kv_begin, kv_end, slot)
    cta_indptr: list
    lists: list  # (req, kvh, qtile, [slots])
    n_slots: int
    image: np.ndarray


def plan_ref(qo_lens, kv_lens, *, g, H_kv, mask=MASK_NONE, num_ctas, tile_set=(16, 64, 128, 256),
             alpha=1, beta=1, align=1, L_min=0, T_q=None, qo_begin=None, page_begin=None, window=0) -> Plan:
    qo_lens = [int(x) for x in qo_lens]
    kv_lens = [int(x) for x in kv_lens]
    B = len(qo_lens)
    if num_ctas < 1:
        raise ValueError("num_ctas >= 1")
    if T_q is None:
        T_q = select_tile(qo_lens, g, tile_set)
    # --- rows (request, kv head, q tile) and their effective kv range [b, e): e is the causal-
    # effective end (R13); with a sliding window W (R26) the tile's first row sees nothing
    # before p - W + 1, so b is that bound rounded down to the chunk alignment
    rows = []  # (i, h, t, b, e)
    for i in range(B):
        lq, lk = qo_lens[i], kv_lens[i]
        fused = lq * g
        for h in range(H_kv):
            for t in range(ceil_div(fused, T_q)):
                if mask == MASK_CAUSAL:
                    hi = min((t + 1) * T_q, fused)
                    last_tok = ceil_div(hi, g) - 1
                    e = min(max(lk - lq + last_tok + 1, 0), lk)
                else:
                    e = lk
                b = 0
                if window > 0:
                    first_tok = (t * T_q) // g
                    b = max(0, lk - lq + first_tok - window + 1)
                    b = min((b // align) * align, e)
                rows.append((i, h, t, b, e))
    total = sum(r[4] - r[3] for r in rows)
    L = max(ceil_div(total, num_ctas), L_min, 1)
    L = ceil_div(L, align) * align
    # --- chunks, work index w in (row, j) order
    chunks = []  # (w, row_idx, j, begin, end)
    for ri, (i, h, t, b, e) in enumerate(rows):
        n = max(1, ceil_div(e - b, L))
        for j in range(n):
            chunks.append((len(chunks), ri, j, b + j * L, min(b + (j + 1) * L, e)))
    # --- slots: DIRECT for unsplit rows, consecutive slots (j asc) for split rows
    nchunk_of_row = [0] * len(rows)
    for c in chunks:
        nchunk_of_row[c[1]] += 1
    slot_of = [-1] * len(chunks)
    lists = []
    nslot = 0
    first_chunk = 0
    for ri, (i, h, t, _b, _e) in enumerate(rows):
        n = nchunk_of_row[ri]
        if n > 1:
            sl = []
            for j in range(n):
                slot_of[first_chunk + j] = nslot
                sl.append(nslot)
                nslot += 1
            lists.append((i, h, t, sl))
        first_chunk += n
    # --- Algorithm 1 lines 5-11: sort desc length (ties: w asc), greedy min-heap
    order = sorted(chunks, key=lambda c: (-(c[4] - c[3]), c[0]))
    heap = [(0, c) for c in range(num_ctas)]
    heapq.heapify(heap)
    queues = [[] for _ in range(num_ctas)]
    for (w, ri, j, b, e) in order:
        cost, cta = heapq.heappop(heap)
        queues[cta].append(w)
        heapq.heappush(heap, (cost + alpha * T_q + beta * (e - b), cta))
    items = []
    cta_indptr = [0]
    for c in range(num_ctas):
        for w in queues[c]:
            _, ri, j, b, e = chunks[w]
            i, h, t, _, _ = rows[ri]
            items.append((i, h, t, b, e, slot_of[w]))
        cta_indptr.append(len(items))
    image = encode_image(num_ctas, T_q, L, items, cta_indptr, lists, nslot, B, g, H_kv, mask, qo_lens,
                         kv_lens, qo_begin, page_begin)
    return Plan(num_ctas, T_q, L, items, cta_indptr, lists, nslot, image)


def encode_image(num_ctas, T_q, L, items, cta_indptr, lists, n_slots, B, g, H_kv, mask, qo_lens, kv_lens,
                 qo_begin=None, page_begin=None) -> np.ndarray:
    """Plan image (int32), the bit-exact contract with the C++ scheduler:
    header[16] = magic, version, num_ctas, T_q, L, n_items, n_lists, n_slots, batch, g, H_kv, mask, 0...
    cta_indptr[num_ctas+1]; item_{req,kvh,qtile,kv_begin,kv_end,slot}[n_items] (queue order);
    list_indptr[n_lists+1]; list_slot[n_slots]; list_{req,kvh,qtile}[n_lists];
    req_{qo_begin,qo_len,kv_len,page_begin}[B]."""
    if qo_begin is None:
        qo_begin = np.concatenate([[0], np.cumsum(qo_lens)])[:B] if B else []
    if page_begin is None:
        page_begin = [0] * B
    hdr = [MAGIC, VERSION, num_ctas, T_q, L, len(items), len(lists), n_slots, B, g, H_kv, mask]
    hdr += [0] * (HEADER_WORDS - len(hdr))
    out = list(hdr) + list(cta_indptr)
    for f in range(6):
        out += [it[f] for it in items]
    li = [0]
    for lst in lists:
        li.append(li[-1] + len(lst[3]))
    out += li
    for lst in lists:
        out += lst[3]
    for f in range(3):
        out += [lst[f] for lst in lists]
    out += [int(x) for x in qo_begin] + list(qo_lens) + list(kv_lens) + [int(x) for x in page_begin]
    return np.array(out, dtype=np.int64).astype(np.int32)


def lengths_from_bsr(qo_indptr, kv_page_indptr, kv_last_page_len, page_size):
    """§8(a) row a1: l_qo(i), l_kv(i) = (n_i-1)*B_c + last_page_len (0 if no pages)."""
    qo_indptr = np.asarray(qo_indptr, np.int64)
    kp = np.asarray(kv_page_indptr, np.int64)
    n = kp[1:] - kp[:-1]
    qo = qo_indptr[1:] - qo_indptr[:-1]
    kv = np.where(n > 0, (n - 1) * page_size + np.asarray(kv_last_page_len, np.int64), 0)
    return qo.astype(np.int64), kv.astype(np.int64)


def cta_costs(plan: Plan, alpha=1, beta=1):
    """Per-CTA cost under the paper's cost model (for balance checks)."""
    c = []
    for k in range(plan.num_ctas):
        s = 0
        for it in plan.items[plan.cta_indptr[k]:plan.cta_indptr[k + 1]]:
            s += alpha * plan.T_q + beta * (it[4] - it[3])
        c.append(s)
    return c
