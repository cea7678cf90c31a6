"""configs[4] long-context decode (4 x 512K, one GPU): per-layer time vs the persistent grid size.
Algorithm 1 cuts each (request, kv head) row into chunks of L = ceil(sum / #CTA) tokens;
with 148 CTAs a row is 4.6 chunks, so the LPT makespan is ~1.6 L. 128 CTAs give exactly 4 chunks
per row. Prints the Algorithm-1 makespan / mean and the measured time for each grid."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402

wl = synth.c5_long_decode()
inp = synth.make_inputs(wl, device="cuda:0")
nq = wl.batch
o = torch.empty((nq, wl.H_qo, wl.D), device="cuda:0")
lse = torch.empty((nq, wl.H_qo), device="cuda:0")
res = {}
for nc in (148, 144, 136, 128, 120):
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, o_dtype="f32",
                           max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=nc, tile_q=16)
    eng = bsra.Engine(cfg, 0)
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    costs, mk = eng.plan_stats()
    run = lambda: eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    for _ in range(3):
        run()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    us = float(np.median(ts)) * 1e3
    kv = int(wl.kv_lens.astype(np.int64).sum()) * wl.H_kv * wl.D * 4
    res[nc] = {"us": round(us, 1), "TB_s": round(kv / us / 1e6, 3), "makespan_over_mean": round(mk / costs.mean(), 3)}
    del eng
print(json.dumps(res))
