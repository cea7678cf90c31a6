"""Quest decode latency vs the persistent grid size: fewer CTAs cut Algorithm 1's
chunks per row (and the fused contraction's merge chain) at the cost of per-SM bandwidth."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402
from bench import time_graph  # noqa: E402

dev = torch.device("cuda:0")
PDL = os.environ.get("QUEST_PDL", "1") == "1"  # 0: launches serialised (latency, no overlap)
for S, P in ((4096, 64), (4096, 256), (32768, 64), (32768, 512)):
    wl, extra = synth.quest_decode(S, P)
    inp = synth.make_inputs(wl, device=dev, extra_pages=extra)
    row = {"workload": f"seq{S}_budget{P}"}
    for nc in (16, 32, 64, 96, 148):
        cfg = bsra.make_config(H_qo=1, H_kv=1, D=128, page_size=16, dtype="bf16", max_batch=wl.batch,
                               max_total_qo_rows=wl.batch, num_ctas=nc, tile_q=16, max_qo_len=1, pdl=PDL)
        e = bsra.Engine(cfg, 0)
        o = torch.empty((wl.batch, 1, 128), device=dev, dtype=torch.bfloat16)
        lse = torch.empty((wl.batch, 1), device=dev)
        e.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
        s = torch.cuda.Stream()

        def twenty():
            for _ in range(20):
                e.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse,
                      stream=s)
        row[nc] = round(time_graph(twenty, s, 10) / 20 * 1e3, 2)
        del e
    print(json.dumps(row), flush=True)
