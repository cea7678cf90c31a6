"""fp8 decode with GQA group 8 (64/8 heads, kC = 8) and 16 (128/8, kC = 16): per-launch time, to
check the register-capped (576-thread) fp8 decode variants. Prints one JSON object."""
import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def timed(wl, reps=11):
    inp = synth.make_inputs(wl, device="cuda:0")
    nq = int(wl.qo_lens.sum())
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                           max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=148, tile_q=16,
                           kv_dtype=wl.kv_dtype or None, k_scale=inp.k_scale, v_scale=inp.v_scale)
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
    return round(float(np.median(ts)) * 1e3, 1)


res = {}
for H in ((64, 8), (128, 8)):
    wl = dataclasses.replace(synth.c2_decode_llama8b(batch=64), H_qo=H[0], H_kv=H[1])
    res[f"{H[0]}/{H[1]}"] = {"bf16_us": timed(wl), "e4m3_us": timed(dataclasses.replace(wl, kv_dtype="e4m3"))}
print(json.dumps(res))
