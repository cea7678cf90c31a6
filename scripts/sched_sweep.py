"""Cost-model / chunk-alignment sweep for the decode plan (configs[1]): Algorithm 1's cost
alpha*T_q + beta*len with alpha in {1..64} (per-item overhead in tokens at T_q = 16)
and chunk alignment 16 (page) or 128 (KV tile). Per variant: tiles per CTA (min/mean/max from the
plan image) and us per launch in a 20-launch PDL graph (the bench's launch mode)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402
from bench import time_graph  # noqa: E402

dev = torch.device("cuda:0")


def tiles_per_cta(img):
    nc, ni = int(img[2]), int(img[5])
    c = 16
    ind = img[c:c + nc + 1]
    c += nc + 1 + 3 * ni
    kb = img[c:c + ni].astype(np.int64)
    ke = img[c + ni:c + 2 * ni].astype(np.int64)
    t = (ke - kb + 127) // 128
    per = np.array([t[ind[i]:ind[i + 1]].sum() for i in range(nc)])
    return [int(per.min()), round(float(per.mean()), 2), int(per.max())], int(ni)


def main():
    wl = synth.c2_decode_llama8b()
    inp = synth.make_inputs(wl, device=dev)
    o = torch.empty((wl.batch, 32, 128), device=dev, dtype=torch.bfloat16)
    lse = torch.empty((wl.batch, 32), device=dev)
    s = torch.cuda.Stream()
    variants = [(a, al, bal) for al in (16, 128) for a in (1, 4, 8, 16, 32, 64) for bal in (False,)]
    variants += [(1, 16, True), (8, 16, True), (8, 128, True)]
    for rep in range(2):
        for a, al, bal in variants:
            cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", max_batch=wl.batch,
                                   max_total_qo_rows=wl.batch, num_ctas=148, tile_q=16, max_qo_len=1, pdl=True,
                                   alpha=a, kv_chunk_align=al, balance_ctas=bal)
            e = bsra.Engine(cfg, 0)
            e.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
            tp, ni = tiles_per_cta(e.export_plan())

            def twenty():
                for _ in range(20):
                    e.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse,
                          stream=s)
            us = time_graph(twenty, s, 10) / 20 * 1e3
            print(json.dumps({"rep": rep, "alpha": a, "align": al, "balance": bal, "items": ni, "tiles_per_cta": tp,
                              "us_per_launch": round(us, 2)}), flush=True)
            del e


if __name__ == "__main__":
    main()
