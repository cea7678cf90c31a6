"""Debug (BSRA_EXPERIMENTS build, abtmp/libbsra_trace.so): per-tile pipeline of CTA 0 of the
tc_decode kernel (clock64, tc_decode.cuh DEC_TTRACE): producer issue (after the stage's empty
wait), MMA sees the stage full, MMA issues S (after s_free), softmax sees S, softmax arrives
p_full; per item the epilogue's o_full and store-done. Prints per-tile rows (cycles relative to
the first producer issue) and medians of load latency, softmax time and tile period."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("BSRA_LIB", os.path.join(ROOT, "abtmp", "libbsra_trace.so"))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")


def run(name, wl, heads, num_ctas):
    inp = synth.make_inputs(wl, device=dev)
    cfg = bsra.make_config(D=128, page_size=16, dtype="bf16", max_batch=wl.batch, max_total_qo_rows=wl.batch,
                           num_ctas=num_ctas, tile_q=16, max_qo_len=1, **heads)
    e = bsra.Engine(cfg, 0)
    o = torch.empty((wl.batch, heads["H_qo"], 128), device=dev, dtype=torch.bfloat16)
    lse = torch.empty((wl.batch, heads["H_qo"]), device=dev)
    e.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    buf = torch.zeros(28 * 1024, dtype=torch.int64, device=dev)
    f = bsra.lib().bsra_debug_set_trace
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    f(e._h, buf.data_ptr())
    for _ in range(3):
        buf.zero_()
        e.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
        torch.cuda.synchronize()
    f(e._h, None)
    t = buf.cpu().numpy().reshape(28, 1024)[20:27].astype(np.float64)
    nt = int((t[0] > 0).sum())
    ni = int((t[5] > 0).sum())
    t0 = t[0, 0]
    rows = []
    for k in range(nt):
        rows.append([int(t[j, k] - t0) if t[j, k] else None for j in range(5)])
    items = [[int(t[5, k] - t0), int(t[6, k] - t0)] for k in range(ni)]
    lat = t[1, :nt] - t[0, :nt]
    smx = t[4, :nt] - t[3, :nt]
    per = np.diff(t[3, :nt])
    s_wait = t[3, :nt] - t[2, :nt]
    print(json.dumps({"workload": name, "ctas": num_ctas, "tiles": nt, "items": ni,
                      "median_load_latency_cyc": float(np.median(lat)), "median_softmax_cyc": float(np.median(smx)),
                      "median_tile_period_cyc": float(np.median(per)) if len(per) else None,
                      "median_S_issue_to_softmax_cyc": float(np.median(s_wait)),
                      "total_cyc": int(max(t[6, :ni].max(), t[4, :nt].max()) - t0)}), flush=True)
    print(json.dumps({"workload": name, "ctas": num_ctas, "tile_rows[issue,full,S,smx_in,smx_out]": rows[:40],
                      "item_rows[o_full,stored]": items[:20]}), flush=True)


if __name__ == "__main__":
    n = 64
    suf = synth.Workload("suf", 32, 8, 128, 16, "bf16", "none", np.ones(n, np.int32), np.full(n, 256, np.int32))
    run("composable_suffix", suf, dict(H_qo=32, H_kv=8), 84)
    run("composable_suffix", suf, dict(H_qo=32, H_kv=8), 148)
    run("c2", synth.c2_decode_llama8b(), dict(H_qo=32, H_kv=8), 148)
