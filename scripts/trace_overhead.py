"""Debug (BSRA_EXPERIMENTS build): where the prefill kernel's fixed cost goes. One item per CTA
(144 CTAs), n KV tiles each; CTA-0 event clocks and every CTA's start / end globaltimer."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
tq = int(sys.argv[2]) if len(sys.argv) > 2 else 256
dev = torch.device("cuda:0")
toks, B = tq // 8, 18
wl = synth.Workload("po", 64, 8, 128, 16, "bf16", "none", np.full(B, toks, np.int32), np.full(B, n * 128, np.int32))
inp = synth.make_inputs(wl, device=dev)
cfg = bsra.make_config(H_qo=64, H_kv=8, D=128, page_size=16, dtype="bf16", max_batch=B, max_total_qo_rows=B * toks,
                       num_ctas=144, tile_q=tq, kv_chunk_min=1 << 20)
eng = bsra.Engine(cfg, 0)
buf = torch.zeros(18 * 1024, dtype=torch.int64, device=dev)
f = bsra.lib().bsra_debug_set_trace
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
f(eng._h, buf.data_ptr())
o = torch.empty((B * toks, 64, 128), device=dev, dtype=torch.bfloat16)
lse = torch.empty((B * toks, 64), device=dev)
eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
for _ in range(3):
    buf.zero_()
    eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(18, 1024)
starts, ends = t[16, :144], t[17, :144]
t0 = starts.min()
ev = {}
for e in range(16):
    nz = np.nonzero(t[e])[0]
    if len(nz):
        ev[e] = [int(x - t[9, 0]) if x else None for x in t[e][:int(nz[-1]) + 1]]
print(json.dumps({"n": n, "T_q": tq, "cta_start_ns_spread": int(starts.max() - t0),
                  "cta_end_ns_min": int(ends.min() - t0), "cta_end_ns_max": int(ends.max() - t0),
                  "cta0_cycles_total": int(t[9, 1] - t[9, 0]), "cta0_events": ev}))
