"""NEXT-2 measurement: configs[1] decode with a bf16 KV cache vs an E4M3 (fp8) KV cache,
per launch (CUDA events, median of 15) on the same lengths, plus the HBM bandwidth each achieves on
its algorithmic bytes (K+V bytes of the visible tokens + q/o/lse/indices). Prints one JSON object."""
import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def timed(wl, reps=15, layers=8):
    """Round-robin over `layers` independent pools so L2 (126 MB) never holds a layer's KV."""
    inps = [synth.make_inputs(wl, device="cuda:0", seed_base=l) for l in range(layers)]
    nq = int(wl.qo_lens.sum())
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
                           max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=148, tile_q=16,
                           kv_dtype=wl.kv_dtype or None, k_scale=inps[0].k_scale, v_scale=inps[0].v_scale)
    eng = bsra.Engine(cfg, 0)
    o = torch.empty((nq, wl.H_qo, wl.D), device="cuda:0", dtype=torch.bfloat16)
    lse = torch.empty((nq, wl.H_qo), device="cuda:0")
    eng.plan(inps[0].qo_indptr, inps[0].kv_page_indptr, inps[0].kv_last_page_len, inps[0].sm_scale)

    def run(i):
        x = inps[i % layers]
        eng.run(x.q, x.k_pool, x.v_pool, x.k_strides, x.v_strides, x.kv_page_indices, o, lse)

    for i in range(layers):
        run(i)
    ts = []
    for r in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run(r)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    us = float(np.median(ts)) * 1e3
    es = 1 if wl.kv_dtype == "e4m3" else 2
    tokens = int(wl.kv_lens.sum())
    kv_bytes = tokens * wl.H_kv * wl.D * 2 * es
    other = nq * wl.H_qo * (wl.D * 2 * 2 + 4) + int(wl.num_pages().sum()) * 4
    return {"us": round(us, 2), "kv_bytes": kv_bytes, "GB_s": round((kv_bytes + other) / us / 1e3, 1),
            "tokens_per_s_per_head": round(tokens * wl.H_kv / us * 1e6 / 1e9, 3), "kernel": eng.selected_kernel()}


c2 = synth.c2_decode_llama8b()
res = {"unit": "us per launch (median of 15, 8 rotating layers > L2); GB_s on algorithmic bytes"}
if not os.environ.get("FP8_ONLY"):
    res["bf16"] = timed(c2)
res["e4m3"] = timed(dataclasses.replace(c2, kv_dtype="e4m3"))
if "bf16" in res:
    res["speedup"] = round(res["bf16"]["us"] / res["e4m3"]["us"], 3)
print(json.dumps(res))
