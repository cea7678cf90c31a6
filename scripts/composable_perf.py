"""configs[3] composable decode: per-layer time of the prefix engine, its contraction, the suffix
engine and the ⊕, and of whole steps for several variants (16 layers, graph replay):
  base       : prefix tiles (64, 128), 148 + 148 CTAs, sequential (round-1 configuration)
  pair       : prefix paired 256-row tiles + queue-count balancing, sequential
  conc_<c>   : pair, prefix on c SMs and suffix on 148 - c SMs concurrently (two streams)"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def graph_ms(fn, s, reps=20):
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):  # replay() launches on the current stream
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    dev = torch.device("cuda:0")
    layers = 16
    cis = [synth.c4_composable(device=dev, seed_base=100 * r) for r in range(layers)]
    c0 = cis[0]
    n = c0.q.shape[0]
    pi = torch.from_numpy(c0.prefix["kv_page_indices"]).to(dev)
    si = torch.from_numpy(c0.suffix["kv_page_indices"]).to(dev)
    outs = [(torch.empty((n, 32, 128), device=dev, dtype=torch.bfloat16), torch.empty((n, 32), device=dev))
            for _ in cis]
    unique = (8192 + n * 256) * 8 * 128 * 4 + n * 32 * 128 * 4 + n * 32 * 4
    s = torch.cuda.Stream()
    res = {}
    variants = [("base", dict(prefix_tiles=(64, 128), balance=False, prefix_ctas=148, suffix_ctas=148)),
                ("pair", dict(prefix_ctas=148, suffix_ctas=148))]
    variants.append(("base_pdl", dict(prefix_tiles=(64, 128), balance=False, prefix_ctas=148, suffix_ctas=148,
                                      pdl=True)))
    variants.append(("pair_pdl", dict(prefix_ctas=148, suffix_ctas=148, pdl=True)))
    for pc, sc in ((56, 92), (64, 84), (72, 76)):
        variants.append((f"conc_{pc}_{sc}", dict(prefix_ctas=pc, suffix_ctas=sc, concurrent=True)))
    variants.append(("pair_pdl_suffix_first", dict(prefix_ctas=148, suffix_ctas=148, pdl=True, suffix_first=True)))
    variants.append(("pair_suffix_first", dict(prefix_ctas=148, suffix_ctas=148, suffix_first=True)))
    variants.append(("conc_64_84_nopdl", dict(prefix_ctas=64, suffix_ctas=84, concurrent=True, pdl=False)))
    variants.append(("conc_64_84_tq128", dict(prefix_ctas=64, suffix_ctas=84, concurrent=True, prefix_tiles=(64, 128))))
    variants.append(("conc_56_92_tq128", dict(prefix_ctas=56, suffix_ctas=92, concurrent=True, prefix_tiles=(64, 128))))
    variants.append(("conc_72_76_tq128", dict(prefix_ctas=72, suffix_ctas=76, concurrent=True, prefix_tiles=(64, 128))))
    variants.append(("conc_64_84_suffix_pdl", dict(prefix_ctas=64, suffix_ctas=84, concurrent=True, pdl=False,
                                                   suffix_pdl=True)))
    variants.append(("conc_64_84_prefix_pdl", dict(prefix_ctas=64, suffix_ctas=84, concurrent=True, pdl=True,
                                                   suffix_pdl=False)))
    for name, kw in variants:
        comp = bsra.ComposableDecode(H_qo=32, H_kv=8, D=128, page_size=16, n_branch=n, **kw)
        comp.plan(c0.prefix, c0.suffix, c0.sm_scale)

        def step():
            for ci, (o, l) in zip(cis, outs):
                comp.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, pi, si, o, l, stream=s)
        ms = graph_ms(step, s) / layers
        # components (sequential, graph of 16 layers each)
        def pre():
            for ci in cis:
                comp.prefix.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, ci.strides, pi, comp.o_p, comp.l_p, stream=s)
        def suf():
            for ci in cis:
                comp.suffix.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, ci.strides, si, comp.o_s, comp.l_s, stream=s)
        def con():
            for (o, l) in outs:
                if comp.fold_suffix:
                    comp.prefix.contract(o, l, o_extra=comp.o_s, lse_extra=comp.l_s, stream=s)
                else:
                    comp.prefix.contract(comp.o_p, comp.l_p, stream=s)
        r = {"us_per_layer": ms * 1e3, "TB/s": unique / (ms * 1e-3) / 1e12,
             "prefix_us": graph_ms(pre, s) / layers * 1e3, "suffix_us": graph_ms(suf, s) / layers * 1e3,
             "contract_us": graph_ms(con, s) / layers * 1e3,
             "prefix_T_q": int(comp.prefix.export_plan()[3]), "prefix_items": int(comp.prefix.export_plan()[5]),
             "prefix_slots": int(comp.prefix.export_plan()[7])}
        res[name] = r
        print(name, json.dumps(r), flush=True)
        del comp
    print(json.dumps(res))


if __name__ == "__main__":
    main()
