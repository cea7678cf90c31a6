"""Debug: configs[1] decode with an E4M3 KV cache (or bf16 with BF16=1), CTA-0 timeline.
Events (clock64 of the SM running CTA 0; index = tile count of that role, items for 6/7):
0 TMA issued, 1 K converter saw fp8 data, 2 K in TMEM, 3 V converted, 4 S ready (softmax),
5 PV issued, 6 item start, 7 item done, 9 kernel start / end. Prints per-event medians of the
inter-tile gaps and the lags between roles."""
import ctypes
import dataclasses
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402

wl = dataclasses.replace(synth.c2_decode_llama8b(), kv_dtype="e4m3")
inp = synth.make_inputs(wl, device="cuda:0")
cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
                       max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=148, tile_q=16,
                       kv_dtype="e4m3", k_scale=inp.k_scale, v_scale=inp.v_scale)
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
t = buf.cpu().numpy().reshape(16, 1024).astype(np.int64)
t0 = t[9, 0]
ev = {}
for e in list(range(9)) + list(range(10, 16)):
    nz = np.nonzero(t[e])[0]
    n = int(nz[-1]) + 1 if len(nz) else 0
    ev[e] = t[e, :n] - t0
res = {"total_cycles": int(t[9, 1] - t0), "tiles": len(ev[0]), "items": len(ev[6])}
for e in range(8):
    if len(ev[e]) > 2:
        res[f"ev{e}_gap_median"] = float(np.median(np.diff(ev[e])))
n = min(len(ev[k]) for k in (0, 1, 2, 3, 4, 5))
if n:
    res["lag_tma_to_data"] = float(np.median(ev[1][:n] - ev[0][:n]))
    res["lag_data_to_K"] = float(np.median(ev[2][:n] - ev[1][:n]))
    res["lag_K_to_Sready"] = float(np.median(ev[4][:n] - ev[2][:n]))
    res["lag_Sready_to_PV"] = float(np.median(ev[5][:n] - ev[4][:n]))
    res["lag_V_to_PV"] = float(np.median(ev[5][:n] - ev[3][:n]))
names = {10: "S_loaded", 11: "p_computed", 12: "pv_waited", 13: "P_stored_fenced", 14: "barrier_passed",
         15: "vfull_waited"}
prev = 4
for e in range(10, 16):
    m = min(len(ev[prev]), len(ev[e]))
    if m:
        res[f"step_{names[e]}"] = float(np.median(ev[e][:m] - ev[prev][:m]))
    prev = e
m = min(len(ev[15]), len(ev[5]))
if m:
    res["step_PV_issued"] = float(np.median(ev[5][:m] - ev[15][:m]))
if len(ev[6]) and len(ev[7]):
    m = min(len(ev[6]), len(ev[7]))
    res["item_span_median"] = float(np.median(ev[7][:m] - ev[6][:m]))
res["first_events"] = {e: [int(x) for x in ev[e][:24]] for e in range(8)}
print(json.dumps(res))
