"""configs[2] causal prefill: plan variants timed as in bench.py (PDL graph of 4 runs over 2
layers): Algorithm 1 at 148 CTAs, with queue-count balancing (BSRA_FLAG_BALANCE_CTAS), and the
cost model's per-item term alpha (cost = alpha * T_q + beta * len)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from bench import Layered, causal_flops, time_graph  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    wl = synth.c3_prefill_llama70b()
    L = Layered(wl, 2, dev)
    fl = causal_flops(wl)
    s = torch.cuda.Stream()
    for rep in range(2):
        for name, kw in (("alg1_148", dict(num_ctas=148)), ("balanced_148", dict(num_ctas=148, balance_ctas=True)),
                         ("alpha8", dict(num_ctas=148, alpha=8)), ("alpha64", dict(num_ctas=148, alpha=64)),
                         ("alpha256", dict(num_ctas=148, alpha=256))):
            e = L.engine(tile_q=0, pdl=True, **kw)
            with torch.cuda.stream(s):
                L.plan(e, s)
            torch.cuda.synchronize()

            def four():
                for r in (0, 1, 0, 1):
                    L.run_layer(e, r, s)
            ms = time_graph(four, s, 5) / 4
            costs, mk = e.plan_stats()
            print(json.dumps({"rep": rep, "variant": name, "ms": round(ms, 4), "TFLOP/s": round(fl / (ms * 1e-3) / 1e12, 1),
                              "cost_eff": round(float(costs.mean() / mk), 4), "items": int(e.export_plan()[5])}),
                  flush=True)
            del e


if __name__ == "__main__":
    main()
