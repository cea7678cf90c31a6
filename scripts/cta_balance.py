"""Debug: per-CTA start/end (globaltimer) of the configs[2] prefill kernel against the plan's
per-CTA work (128-token KV tiles, visible-pair cost), to separate load imbalance from per-tile
speed. Usage: python scripts/cta_balance.py T_q [T_q ...]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_01005_b200 as bsra  # noqa: E402
import synth  # noqa: E402

wl = synth.c2_decode_llama8b() if os.environ.get("DECODE") else synth.c3_prefill_llama70b()
inp = synth.make_inputs(wl, device="cuda:0")
nq = int(inp.qo_indptr[-1])
for tq in [int(x) for x in sys.argv[1:]] or [128, 256]:  # DECODE=1: configs[1] with T_q = 16
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
                           max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()), num_ctas=148, tile_q=tq)
    eng = bsra.Engine(cfg, 0)
    buf = torch.zeros(20 * 1024, dtype=torch.int64, device="cuda:0")
    f = bsra.lib().bsra_debug_set_trace
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    f(eng._h, buf.data_ptr())
    o = torch.empty((nq, wl.H_qo, wl.D), device="cuda:0", dtype=torch.bfloat16)
    lse = torch.empty((nq, wl.H_qo), device="cuda:0")
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    for _ in range(3):
        buf.zero_()
        eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    torch.cuda.synchronize()
    t = buf.cpu().numpy().reshape(20, 1024)
    st, en = t[16, :148].astype(np.float64), t[17, :148].astype(np.float64)
    t0 = st.min()
    st, en = (st - t0) / 1e3, (en - t0) / 1e3  # us
    dur = en - st
    im = eng.export_plan()
    nc, n_items = int(im[2]), int(im[5])
    cta = im[16:16 + nc + 1]
    base = 16 + nc + 1
    kb = im[base + 3 * n_items: base + 4 * n_items].astype(np.int64)
    ke = im[base + 4 * n_items: base + 5 * n_items].astype(np.int64)
    tiles = np.array([int(np.sum((ke[cta[c]:cta[c + 1]] - kb[cta[c]:cta[c + 1]] + 127) // 128)) for c in range(nc)])
    toks = np.array([int(np.sum(ke[cta[c]:cta[c + 1]] - kb[cta[c]:cta[c + 1]])) for c in range(nc)])
    items = np.diff(cta)
    costs, _ = eng.plan_stats()
    us_per_tile = dur / np.maximum(tiles, 1)
    print(f"T_q={tq}: kernel {en.max():.1f} us; start skew max {st.max():.1f} us; CTA dur min/med/max "
          f"{dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us")
    print(f"   tiles/CTA min/med/max {tiles.min()}/{int(np.median(tiles))}/{tiles.max()}  items/CTA "
          f"{items.min()}/{int(np.median(items))}/{items.max()}  cost min/max {costs.min()}/{costs.max()}")
    print(f"   tokens/CTA min/med/max {toks.min()}/{int(np.median(toks))}/{toks.max()}; "
          f"GB/s per CTA med {np.median(toks * 512 / dur / 1e3):.1f}; whole kernel {toks.sum() * 512 / en.max() / 1e3:.0f} GB/s")
    print(f"   us/tile min/med/max {us_per_tile.min():.3f}/{np.median(us_per_tile):.3f}/{us_per_tile.max():.3f}; "
          f"corr(dur, tiles) {np.corrcoef(dur, tiles)[0, 1]:.3f}; corr(dur, items) {np.corrcoef(dur, items)[0, 1]:.3f}")
    order = np.argsort(dur)
    for c in list(order[:3]) + list(order[-3:]):
        print(f"   cta {c:3d}: start {st[c]:7.1f} end {en[c]:7.1f} tiles {tiles[c]:4d} items {items[c]:3d} cost {costs[c]}")
