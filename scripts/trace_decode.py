"""Debug (BSRA_EXPERIMENTS build, abtmp/libbsra_trace.so): where a tc_decode launch's fixed cost
goes. Per CTA globaltimer events (tc_decode.cuh DEC_TRACE): 7 kernel entry, 0 plan staged,
6 setup done, 1 first S^T ready (first K landed), 2 softmax done, 3 epilogue past pdl_wait,
4 last item's o stored, 5 contraction done, 17 end. Prints per-event [min, median, max] in ns
relative to the earliest kernel entry, and the event-timed launch (us) alone and in a 20-launch
graph (with / without PDL)."""
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
from bench import time_graph  # noqa: E402

dev = torch.device("cuda:0")
EV = [(7, "entry"), (0, "staged"), (6, "setup"), (11, "producer_start"), (8, "first_kv_issue"), (9, "mma_q_full"),
      (10, "mma_kv0_full"), (1, "first_S"), (2, "softmax_done"), (3, "pdl_wait"),
      (4, "last_o"), (5, "contr_done"), (17, "end")]


def workloads():
    wl, extra = synth.quest_decode(4096, 64)
    yield "quest4096_64", wl, extra, dict(H_qo=1, H_kv=1)
    n = 64
    yield "composable_suffix", synth.Workload("suf", 32, 8, 128, 16, "bf16", "none", np.ones(n, np.int32),
                                              np.full(n, 256, np.int32)), 0, dict(H_qo=32, H_kv=8)
    yield "c2", synth.c2_decode_llama8b(), 0, dict(H_qo=32, H_kv=8)


def one(name, wl, extra, heads, num_ctas=148, pdl=False, dump=False):
    inp = synth.make_inputs(wl, device=dev, extra_pages=extra)
    cfg = bsra.make_config(D=128, page_size=16, dtype="bf16", max_batch=wl.batch, max_total_qo_rows=wl.batch,
                           num_ctas=num_ctas, tile_q=16, max_qo_len=1, pdl=pdl, **heads)
    e = bsra.Engine(cfg, 0)
    o = torch.empty((wl.batch, heads["H_qo"], 128), device=dev, dtype=torch.bfloat16)
    lse = torch.empty((wl.batch, heads["H_qo"]), device=dev)
    e.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    s = torch.cuda.Stream()

    def run():
        e.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse, stream=s)

    def twenty():
        for _ in range(20):
            run()
    g_us = time_graph(twenty, s, 10) / 20 * 1e3
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(9):
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            a.record(s)
            run()
            b.record(s)
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) * 1e3)
    buf = torch.zeros(18 * 1024, dtype=torch.int64, device=dev)
    f = bsra.lib().bsra_debug_set_trace
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    f(e._h, buf.data_ptr())
    res = []
    for _ in range(3):
        buf.zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            run()
        torch.cuda.synchronize()
        t = buf.cpu().numpy().reshape(18, 1024)[:, :num_ctas].astype(np.float64)
        if not (t[7] > 0).any():  # not a BSRA_EXPERIMENTS build: timings only
            res.append({})
            continue
        t0 = t[7][t[7] > 0].min()
        row = {}
        for ev, nm in EV:
            x = t[ev][t[ev] > 0] - t0
            if len(x):
                row[nm] = [int(x.min()), int(np.median(x)), int(x.max())]
        res.append(row)
    f(e._h, None)
    if not res[-1]:
        print(json.dumps({"workload": name, "pdl": pdl, "ctas": num_ctas, "graph20_us": g_us,
                          "launch_us_median": float(np.median(times))}))
        return
    # per CTA: tiles in its queue (plan image), SM id, first-S and softmax-done times
    img = e.export_plan()
    nc = int(img[2]); ni = int(img[5])
    c = 16
    cta_indptr = img[c:c + nc + 1]; c += nc + 1
    c += 3 * ni
    kb = img[c:c + ni].astype(np.int64); c += ni
    ke = img[c:c + ni].astype(np.int64)
    tiles = (ke - kb + 127) // 128
    per = [int(tiles[cta_indptr[i]:cta_indptr[i + 1]].sum()) for i in range(nc)]
    sm = t[15].astype(np.int64) - 1
    done = t[2] - t0
    first = t[1] - t0
    order = np.argsort(done)
    cta_rows = [[int(i), per[i], int(sm[i]), int(first[i]), int(done[i])] for i in order]
    tp = np.array(per, np.float64)
    d = done.astype(np.float64)
    ok = d > 0
    corr = float(np.corrcoef(tp[ok], d[ok])[0, 1]) if ok.sum() > 2 and tp[ok].std() > 0 else None
    print(json.dumps({"workload": name, "pdl": pdl, "ctas": num_ctas,
                      "launch_us_median": float(np.median(times)), "graph20_us": g_us, "trace_ns": res[-1],
                      "tiles_per_cta": [int(tp.min()), float(tp.mean()), int(tp.max())], "corr_tiles_done": corr}))
    if dump:
        print(json.dumps({"workload": name, "cta_tiles_sm_first_done_sorted": cta_rows}))


if __name__ == "__main__":
    for name, wl, extra, heads in workloads():
        for pdl in (False, True):
            one(name, wl, extra, heads, pdl=pdl, dump=(name == "c2" and not pdl))
