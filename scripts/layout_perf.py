"""configs[1] decode per-launch time for the pool layouts NHD [pages, B_c, H_kv, D] and
HND [pages, H_kv, B_c, D] (both are BSR page pools the paper's API accepts), and for
page sizes 16 / 32 / 64 (median of 9 launches, CUDA events)."""
import dataclasses
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from tests.helpers import engine_for  # noqa: E402


def timed(fn, reps=9):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3


def main():
    dev = torch.device("cuda:0")
    res = {}
    base = synth.c2_decode_llama8b()
    for ps in (16, 32, 64):
        for layout in ("NHD", "HND"):
            wl = dataclasses.replace(base, page_size=ps)
            inp = synth.make_inputs(wl, device=dev, layout=layout)
            eng = engine_for(wl, num_ctas=148, tile_q=16)
            o = torch.empty((wl.batch, wl.H_qo, wl.D), device=dev, dtype=torch.bfloat16)
            lse = torch.empty((wl.batch, wl.H_qo), device=dev)
            eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
            us = timed(lambda: eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides,
                                       inp.kv_page_indices, o, lse))
            kv = int(wl.kv_lens.sum()) * 8 * 128 * 4
            res[f"ps{ps}_{layout}"] = {"us": us, "kv_TB/s": kv / (us * 1e-6) / 1e12}
            print(ps, layout, round(us, 1), flush=True)
            del inp, eng
            torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
