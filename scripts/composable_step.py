"""configs[3] composable step, eager (no graph) so a profiler sees every launch: the bench's
configuration (prefix engine on 64 SMs concurrently with the suffix engine on 84, then one
bsra_contract launch folding prefix slots and suffix state). Runs `reps` layers.
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/composable_step.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def main(reps=4):
    dev = torch.device("cuda:0")
    ci = synth.c4_composable(device=dev)
    n = ci.q.shape[0]
    comp = bsra.ComposableDecode(H_qo=32, H_kv=8, D=128, page_size=16, n_branch=n, prefix_ctas=64, suffix_ctas=84,
                                 concurrent=True)
    comp.plan(ci.prefix, ci.suffix, ci.sm_scale)
    pi = torch.from_numpy(ci.prefix["kv_page_indices"]).to(dev)
    si = torch.from_numpy(ci.suffix["kv_page_indices"]).to(dev)
    o = torch.empty((n, 32, 128), device=dev, dtype=torch.bfloat16)
    lse = torch.empty((n, 32), device=dev)
    for _ in range(reps):
        comp.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, pi, si, o, lse)
    torch.cuda.synchronize()
    print("launches per layer:", comp.launches())


if __name__ == "__main__":
    main()
