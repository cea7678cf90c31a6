"""NEXT-3 measurement: per-launch time of the attention variants on the BASELINE configs
(CUDA events, median of 9): configs[1] decode with sliding windows (the plan reads only the
window, so time should follow the keys read) and configs[2] prefill with a window and with a
logits soft-cap. Prints one JSON object."""
import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def timed(wl, tile_q, reps=9):
    inp = synth.make_inputs(wl, device="cuda:0")
    nq = int(wl.qo_lens.sum())
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
                           max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=148, tile_q=tile_q, window=wl.window,
                           soft_cap=wl.soft_cap)
    eng = bsra.Engine(cfg, 0)
    o = torch.empty((nq, wl.H_qo, wl.D), device="cuda:0", dtype=torch.bfloat16)
    lse = torch.empty((nq, wl.H_qo), device="cuda:0")
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    run = lambda: eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    for _ in range(3):
        run()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    im = eng.export_plan()
    n_items, base = int(im[5]), 16 + int(im[2]) + 1
    keys = int((im[base + 4 * n_items: base + 5 * n_items] - im[base + 3 * n_items: base + 4 * n_items]).sum())
    return {"us": round(float(np.median(ts)) * 1e3, 2), "keys_read": keys}


c2, c3 = synth.c2_decode_llama8b(), synth.c3_prefill_llama70b()
res = {"unit": "us per launch (median of 9); keys_read = sum of the plan's item ranges (x kv heads)"}
res["decode_c2"] = {f"window_{w}" if w else "full": timed(dataclasses.replace(c2, window=w), 16)
                    for w in (0, 4096, 1024, 256)}
res["decode_c2"]["soft_cap_50"] = timed(dataclasses.replace(c2, soft_cap=50.0), 16)
res["prefill_c3"] = {"full": timed(c3, 0), "window_1024": timed(dataclasses.replace(c3, window=1024), 0),
                     "soft_cap_50": timed(dataclasses.replace(c3, soft_cap=50.0), 0)}
print(json.dumps(res))
