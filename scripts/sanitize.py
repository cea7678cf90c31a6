"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): CUDA-core decode (configs[0], split across 4 CTAs => contraction),
tcgen05 decode (kC 4 and 16, split + fused contraction, PDL), tcgen05 prefill (streamed and
paired tiles, causal + custom mask), fp8 decode and the fp8 gather + prefill path, contiguous
KV, merge kernels. Each case is checked against the oracle so a run also proves the results.

  compute-sanitizer --tool memcheck python scripts/sanitize.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402
from tests.helpers import assert_close, run_gpu  # noqa: E402


def main():
    # --no-cp-async: leave out the cp.async row-gather case (racecheck does not model the tensor
    # core's commit barrier that orders a stage's reuse)
    skip_cp = "--no-cp-async" in sys.argv
    dev = torch.device("cuda:0")
    W = synth.Workload
    cases = [
        ("simt c1 split", synth.c1_tiny_decode(), dict(num_ctas=4)),
        ("tc_decode kC4 split", W("d", 32, 8, 128, 16, "bf16", "none", np.ones(3, np.int32),
                                  np.array([700, 33, 300], np.int32)), dict(num_ctas=8, tile_q=16)),
        ("tc_decode kC16 causal", W("d", 32, 8, 128, 16, "bf16", "causal", np.array([4, 1], np.int32),
                                    np.array([300, 129], np.int32)), dict(num_ctas=5, tile_q=16)),
        ("tc_prefill streamed causal", W("p", 64, 8, 128, 16, "bf16", "causal", np.array([70, 130], np.int32),
                                         np.array([70, 200], np.int32)), dict(num_ctas=6, tile_q=128)),
        ("tc_prefill paired custom", W("p", 64, 8, 128, 16, "bf16", "custom", np.array([40, 9], np.int32),
                                       np.array([300, 9], np.int32)), dict(num_ctas=5, tile_q=256)),
        ("tc_decode fp8", W("f", 32, 8, 128, 16, "bf16", "none", np.ones(2, np.int32),
                            np.array([300, 17], np.int32), kv_dtype="e4m3"), dict(num_ctas=4, tile_q=16)),
        ("fp8 gather + prefill", W("f", 64, 8, 128, 16, "bf16", "causal", np.array([70, 1], np.int32),
                                   np.array([70, 300], np.int32), kv_dtype="e4m3"), dict(num_ctas=4, tile_q=128)),
        ("tc_decode RoPE", W("r", 32, 8, 128, 16, "bf16", "causal", np.array([1, 3], np.int32),
                             np.array([300, 70], np.int32), rope_theta=10000.0), dict(num_ctas=6, tile_q=16)),
        ("tc_decode gather4 B_c=1", W("g", 32, 8, 128, 1, "bf16", "none", np.ones(2, np.int32),
                                      np.array([200, 33], np.int32)), dict(num_ctas=4, tile_q=16)),
        ("tc_decode cp.async B_c=4", W("c", 32, 8, 128, 4, "bf16", "none", np.ones(2, np.int32),
                                       np.array([200, 33], np.int32)), dict(num_ctas=4, tile_q=16, cp_async=True)),
        ("simt RoPE prefill", W("s", 32, 8, 128, 16, "bf16", "causal", np.array([20, 1], np.int32),
                                np.array([20, 90], np.int32), rope_theta=10000.0), dict(num_ctas=4, tile_q=64)),
    ]
    if skip_cp:
        cases = [c for c in cases if "cp.async" not in c[0]]
    if "--only-cp-async" in sys.argv:
        cases = [c for c in cases if "cp.async" in c[0]]
    for name, wl, kw in cases:
        inp = synth.make_inputs(wl, device=dev)
        gpu = run_gpu(inp, **kw)
        do, dl = assert_close(gpu, oracle.attention_from_inputs(inp), wl.dtype, what=name)
        print(f"ok {name}: kernel={gpu[2].selected_kernel()} max|do|={do:.3g} max|dlse|={dl:.3g}", flush=True)
    # merge kernels
    g = torch.Generator().manual_seed(1)
    oa, ob = torch.rand((5, 4, 128), generator=g).to(dev), torch.rand((5, 4, 128), generator=g).to(dev)
    la, lb = torch.randn((5, 4), generator=g).to(dev), torch.randn((5, 4), generator=g).to(dev)
    bsra.merge_states(oa, la, ob, lb)
    op = torch.rand((3, 5, 4, 128), generator=g).to(dev)
    lp = torch.randn((3, 5, 4), generator=g).to(dev)
    bsra.merge_many(op, lp, torch.empty((5, 4, 128), device=dev), torch.empty((5, 4), device=dev))
    torch.cuda.synchronize()
    print("ok merge kernels", flush=True)


if __name__ == "__main__":
    main()
