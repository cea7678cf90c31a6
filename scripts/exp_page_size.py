"""Timing experiment: does the TMA box size (= page size, up to 128 tokens) bound the kernels?
Runs configs[1] decode and configs[2] prefill at page sizes 16 / 32 / 64 / 128 (same lengths,
permuted pages) and prints per-launch times (CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def time_run(wl, tile_q, reps=5, **kw):
    inp = synth.make_inputs(wl, device="cuda:0")
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                           mask=wl.mask, max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=148,
                           tile_q=tile_q, **kw)
    eng = bsra.Engine(cfg, 0)
    nq = int(inp.qo_indptr[-1])
    o = torch.empty((nq, wl.H_qo, wl.D), device="cuda:0", dtype=torch.bfloat16)
    lse = torch.empty((nq, wl.H_qo), device="cuda:0")
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    for _ in range(2):
        eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3


for ps in (16, 32, 64, 128):
    c2 = synth.c2_decode_llama8b()
    c2.page_size = ps
    c3 = synth.c3_prefill_llama70b()
    c3.page_size = ps
    print(f"page {ps:4d}: decode {time_run(c2, 16):8.1f} us   prefill {time_run(c3, 128):8.1f} us", flush=True)
