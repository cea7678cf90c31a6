"""Prefill kernel fixed cost vs per-tile cost: 148 requests x 8 kv heads' worth of tiles, one item
per CTA (num_ctas = rows, no split), each with n KV tiles of 128 tokens; per-launch time (median of
7) for n in {1, 2, 4, 8, 16, 32} at T_q = 128 and 256 (mask none, 64/8 heads)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def timed(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3


dev = torch.device("cuda:0")
for tq in (128, 256):
    toks = tq // 8  # query tokens per request: one q tile per (request, kv head)
    B = 18  # 18 requests x 8 kv heads = 144 rows = 144 CTAs, one item each
    for n in (1, 2, 4, 8, 16, 32):
        wl = synth.Workload("po", 64, 8, 128, 16, "bf16", "none", np.full(B, toks, np.int32),
                            np.full(B, n * 128, np.int32))
        inp = synth.make_inputs(wl, device=dev)
        cfg = bsra.make_config(H_qo=64, H_kv=8, D=128, page_size=16, dtype="bf16", max_batch=B,
                               max_total_qo_rows=B * toks, num_ctas=144, tile_q=tq, kv_chunk_min=1 << 20)
        eng = bsra.Engine(cfg, 0)
        o = torch.empty((B * toks, 64, 128), device=dev, dtype=torch.bfloat16)
        lse = torch.empty((B * toks, 64), device=dev)
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
        us = timed(lambda: eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices,
                                   o, lse))
        flops = 4.0 * 128 * 64 * B * toks * n * 128
        print(f"T_q={tq} tiles/CTA={n}: {us:.1f} us  {flops / us / 1e6:.0f} TFLOP/s", flush=True)
        del inp, eng, o, lse
