"""Timing experiment: configs[2] causal prefill per-launch time (CUDA events, median of 5) for the
library BSRA_LIB points at. Usage: python scripts/ab_prefill.py T_q [T_q ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def causal_flops(wl):
    vis = 0
    for lq, lk in zip(wl.qo_lens.tolist(), wl.kv_lens.tolist()):
        vis += sum(min(lk, lk - lq + r + 1) for r in range(lq))
    return 4.0 * wl.D * wl.H_qo * vis


wl = synth.c3_prefill_llama70b()
wl.page_size = int(os.environ.get("PAGE", wl.page_size))  # timing experiment: TMA box = page
inp = synth.make_inputs(wl, device="cuda:0")
fl = causal_flops(wl)
for tq in [int(x) for x in sys.argv[1:]] or [128]:
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
                           max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=148,
                           tile_set=(16, 64, 128) if tq <= 128 else (16, 64, 128, 256), tile_q=tq)
    eng = bsra.Engine(cfg, 0)
    nq = int(inp.qo_indptr[-1])
    o = torch.empty((nq, wl.H_qo, wl.D), device="cuda:0", dtype=torch.bfloat16)
    lse = torch.empty((nq, wl.H_qo), device="cuda:0")
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
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
    ms = float(np.median(ts))
    print(f"{os.path.basename(os.environ.get('BSRA_LIB', 'libbsra.so'))} page={wl.page_size} T_q={tq}: {ms * 1e3:.1f} us "
          f"{fl / ms / 1e9:.1f} TFLOP/s", flush=True)
