"""SURVEY §8(f) NEXT-1 study: the cost of the page table on B200 (the paper's App. B ablation,
P:425-447: <= 1 % for decode, ~10 % for prefill on FA3, whose sparse loads could not use TMA).
Same keys / values, three layouts: paged with permuted pages (the workload's scattered pool),
paged with pages in order, and contiguous (ragged) KV with no page table. Per-launch CUDA-event
time (median of 9) for configs[1] decode (T_q = 16) and configs[2] causal prefill (T_q = 256).
Prints one JSON object."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=9):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3


def study(wl, tile_q):
    nq = int(wl.qo_lens.sum())
    out = {}
    for name, permute in (("paged_permuted", True), ("paged_in_order", False)):
        inp = synth.make_inputs(wl, device="cuda:0", permute=permute)
        cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                               mask=wl.mask, max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=148, tile_q=tile_q)
        eng = bsra.Engine(cfg, 0)
        o = torch.empty((nq, wl.H_qo, wl.D), device="cuda:0", dtype=torch.bfloat16)
        lse = torch.empty((nq, wl.H_qo), device="cuda:0")
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
        out[name] = timed(lambda: eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides,
                                          inp.kv_page_indices, o, lse))
        if permute:
            rk = synth.ragged_kv(inp)
            rcfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=128, dtype=wl.dtype, mask=wl.mask,
                                    max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=148, tile_q=tile_q,
                                    ragged_kv=True)
            reng = bsra.Engine(rcfg, 0)
            reng.plan_ragged(inp.qo_indptr, rk.kv_indptr, inp.sm_scale)
            o2 = torch.empty_like(o)
            out["contiguous"] = timed(lambda: reng.run_ragged(inp.q, rk.k, rk.v, rk.k_strides, rk.v_strides, o2,
                                                              lse))
            torch.cuda.synchronize()
            out["max_abs_diff_contiguous_vs_paged"] = float((o2.float() - o.float()).abs().max())
            del rk, reng
        del inp, eng
        torch.cuda.empty_cache()
    out = {k: round(v, 2) if isinstance(v, float) else v for k, v in out.items()}
    out["page_table_overhead_pct"] = round(100.0 * (out["paged_permuted"] / out["contiguous"] - 1.0), 2)
    return out


res = {"unit": "us per launch (CUDA events, median of 9)",
       "decode_c2": study(synth.c2_decode_llama8b(), 16),
       "prefill_c3": study(synth.c3_prefill_llama70b(), 256)}
print(json.dumps(res))
