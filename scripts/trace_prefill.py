"""Debug: run configs[2] prefill once with CTA-0 pipeline tracing and dump the event timeline.
Events (clock64 of SM running CTA 0): 0 K TMA issued (pos), 1 V TMA issued (pos),
2 MMA S issued (pos), 3 MMA PV issued (pv pos), 4 MMA got V (pv pos), 5/6 WG0 S-ready / P-ready,
7/8 WG1 S-ready / P-ready (WG-local tile count), 9 kernel start/end."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402

wl = synth.c3_prefill_llama70b()
inp = synth.make_inputs(wl, device="cuda:0")
cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
                       max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=148)
eng = bsra.Engine(cfg, 0)
buf = torch.zeros(16 * 1024, dtype=torch.int64, device="cuda:0")
f = bsra.lib().bsra_debug_set_trace
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
f(eng._h, buf.data_ptr())
nq = int(inp.qo_indptr[-1])
o = torch.empty((nq, wl.H_qo, wl.D), device="cuda:0", dtype=torch.bfloat16)
lse = torch.empty((nq, wl.H_qo), device="cuda:0")
eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
for _ in range(3):
    buf.zero_()
    eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(16, 1024)
t0 = t[9, 0]
out = {}
for ev in range(16):
    row = t[ev]
    nz = np.nonzero(row)[0]
    n = int(nz[-1]) + 1 if len(nz) else 0
    out[ev] = [int(x - t0) if x else None for x in row[:n]]
print(json.dumps({"total": int(t[9, 1] - t0), "events": out}))
