"""Debug (BSRA_EXPERIMENTS build, abtmp/libbsra_trace.so): timeline of one configs[3] composable
layer inside a CUDA graph (the 2nd of 2 layers is traced): per kernel the [first CTA start,
median, last CTA end] in ns relative to the prefix kernel's first CTA start (globaltimer), so the
gaps between launches and each kernel's in-CTA window show. Prefix = tc_prefill (events 16/17),
suffix = tc_decode (events 7 entry / 5 epilogue done)."""
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


def main():
    dev = torch.device("cuda:0")
    cis = [synth.c4_composable(device=dev, seed_base=100 * r) for r in range(2)]
    c0 = cis[0]
    n = c0.q.shape[0]
    pi = torch.from_numpy(c0.prefix["kv_page_indices"]).to(dev)
    si = torch.from_numpy(c0.suffix["kv_page_indices"]).to(dev)
    outs = [(torch.empty((n, 32, 128), device=dev, dtype=torch.bfloat16), torch.empty((n, 32), device=dev))
            for _ in cis]
    s = torch.cuda.Stream()
    f = bsra.lib().bsra_debug_set_trace
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    for name, kw in (("seq", dict(prefix_ctas=148, suffix_ctas=148)),
                     ("seq_pdl", dict(prefix_ctas=148, suffix_ctas=148, pdl=True)),
                     ("conc_64_84", dict(prefix_ctas=64, suffix_ctas=84, concurrent=True))):
        comp = bsra.ComposableDecode(H_qo=32, H_kv=8, D=128, page_size=16, n_branch=n, **kw)
        comp.plan(c0.prefix, c0.suffix, c0.sm_scale)
        bp = torch.zeros(18 * 1024, dtype=torch.int64, device=dev)
        bs = torch.zeros(18 * 1024, dtype=torch.int64, device=dev)
        f(comp.prefix._h, bp.data_ptr())
        f(comp.suffix._h, bs.data_ptr())

        def step():
            for ci, (o, l) in zip(cis, outs):
                comp.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, pi, si, o, l, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        for _ in range(3):
            with torch.cuda.stream(s):
                g.replay()
            torch.cuda.synchronize()
        tp = bp.cpu().numpy().reshape(18, 1024).astype(np.float64)
        ts = bs.cpu().numpy().reshape(18, 1024).astype(np.float64)
        ncp = comp.prefix.export_plan()[2]
        ncs = comp.suffix.export_plan()[2]
        p_st, p_en = tp[16, :ncp], tp[17, :ncp]
        s_st, s_en = ts[7, :ncs], ts[5, :ncs]
        s_first = ts[1, :ncs]
        t0 = p_st[p_st > 0].min()

        def rng(x):
            x = x[x > 0] - t0
            return [int(x.min()), int(np.median(x)), int(x.max())] if len(x) else None
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            for _ in range(10):
                g.replay()
            b.record(s)
        torch.cuda.synchronize()
        print(json.dumps({"variant": name, "us_per_layer_traced_build": a.elapsed_time(b) / 10 / 2 * 1e3,
                          "prefix_start": rng(p_st), "prefix_end": rng(p_en), "suffix_start": rng(s_st),
                          "suffix_first_S": rng(s_first), "suffix_end": rng(s_en),
                          "prefix_T_q": int(comp.prefix.export_plan()[3]),
                          "prefix_items": int(comp.prefix.export_plan()[5])}), flush=True)
        f(comp.prefix._h, None)
        f(comp.suffix._h, None)
        del comp, g


if __name__ == "__main__":
    main()
