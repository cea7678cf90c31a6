"""configs[3] composable: run the prefix engine, its contraction and the suffix engine a few times
(one layer) so `ncu --metrics gpu__time_duration.sum` lists each kernel's duration."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
c0 = synth.c4_composable(device=dev)
n = c0.q.shape[0]
pi = torch.from_numpy(c0.prefix["kv_page_indices"]).to(dev)
si = torch.from_numpy(c0.suffix["kv_page_indices"]).to(dev)
tiles = (64, 128) if len(sys.argv) > 1 and sys.argv[1] == "t128" else (64, 128, 256)
comp = bsra.ComposableDecode(H_qo=32, H_kv=8, D=128, page_size=16, n_branch=n, prefix_ctas=148, suffix_ctas=148,
                             prefix_tiles=tiles)
comp.plan(c0.prefix, c0.suffix, c0.sm_scale)
o = torch.empty((n, 32, 128), device=dev, dtype=torch.bfloat16)
l = torch.empty((n, 32), device=dev)
for _ in range(4):
    comp.run(c0.q, c0.k_pool, c0.v_pool, c0.strides, pi, si, o, l)
torch.cuda.synchronize()
im = comp.prefix.export_plan()
print("prefix T_q", im[3], "items", im[5], "lists", im[6], "slots", im[7], "L", im[4])
