"""Full-size parity in the bench's own launch configurations (VERDICT r1 "untested configs"):

* configs[4] (4 x 512K tokens, 32/8 heads): one 512K request, all 32 qo heads, element by element
  against the float64 oracle, under the bench's engine (148 CTAs, BSRA_FLAG_BALANCE_CTAS, fp32
  state) with the library's NCCL all-gather + merge on one rank, and with 4 simulated sequence
  shards merged by bsra_merge_many. This is the long-accumulation case SURVEY §8(c.5) warns
  about (a 512K row must not be summed serially in one fp32 register).
* the headline graph: 4 configs[1] layers (each its own q / pools / o, one page table), PDL,
  148 CTAs, max_qo_len 1, captured once and replayed twice; layers 1 and 3 checked on every row.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2501_01005_b200 as bsra
import synth
from tests.helpers import assert_close, rows_of_requests

pytestmark = pytest.mark.gpu


def _c5_engine(wl, nq, local=0):
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                           o_dtype="f32", max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=148, tile_q=16,
                           balance_ctas=True)
    return bsra.Engine(cfg, local)


def test_c5_full_size_one_request_all_heads(cuda_device):
    wl = synth.c5_long_decode()
    inp = synth.make_inputs(wl, device=cuda_device)
    nq = wl.batch
    ref = oracle.attention_from_inputs(synth.request_subset(inp, [0]))  # request 0: 512K tokens, 32 heads
    # (a) P = 1 exactly as bench_long_context: fp32 state, then bsra_dist all-gather + merge
    eng = _c5_engine(wl, nq)
    o_loc = torch.empty((nq, wl.H_qo, wl.D), device=cuda_device)
    l_loc = torch.empty((nq, wl.H_qo), device=cuda_device)
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o_loc, l_loc)
    d = bsra.Dist(1, 0, bsra.Dist.unique_id(), 0)
    scratch = d.scratch(nq, wl.H_qo, wl.D, cuda_device)
    o = torch.empty((nq, wl.H_qo, wl.D), device=cuda_device, dtype=torch.bfloat16)
    l = torch.empty((nq, wl.H_qo), device=cuda_device)
    d.allgather_merge(o_loc, l_loc, scratch, o, l)
    d.check()
    torch.cuda.synchronize()
    d.close()
    assert_close((o[:1].float().cpu().numpy(), l[:1].cpu().numpy()), ref, "bf16", what="c5 P=1 (NCCL merge)")
    # the plan really split the row (otherwise this would not test the contraction)
    img = eng.export_plan()
    assert img[7] > 0, "no partial slots: the 512K rows were not split"
    # (b) 4 simulated sequence shards (bsra_dist_shard_bsr) merged in rank order
    P = 4
    idx = inp.kv_page_indices.cpu().numpy()
    o_parts = torch.empty((P, nq, wl.H_qo, wl.D), device=cuda_device)
    l_parts = torch.empty((P, nq, wl.H_qo), device=cuda_device)
    for r in range(P):
        ki, kx, kl = bsra.sequence_shard(inp.kv_page_indptr, idx, inp.kv_last_page_len, wl.page_size, P, r)
        e = _c5_engine(wl, nq)
        e.plan(inp.qo_indptr, ki, kl, inp.sm_scale)
        e.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, torch.from_numpy(kx).to(cuda_device),
              o_parts[r], l_parts[r])
    o4 = torch.empty((nq, wl.H_qo, wl.D), device=cuda_device, dtype=torch.bfloat16)
    l4 = torch.empty((nq, wl.H_qo), device=cuda_device)
    bsra.merge_many(o_parts, l_parts, o4, l4)
    torch.cuda.synchronize()
    assert_close((o4[:1].float().cpu().numpy(), l4[:1].cpu().numpy()), ref, "bf16", what="c5 P=4 simulated")


def test_headline_graph_four_layers(cuda_device):
    wl = synth.c2_decode_llama8b()
    layers = []
    for r in range(4):
        inp = synth.make_inputs(wl, device=cuda_device, seed_base=100 * r)
        if r > 0:
            inp.kv_page_indices = layers[0][0].kv_page_indices  # one page table per model
        o = torch.full((wl.batch, wl.H_qo, wl.D), float("nan"), device=cuda_device, dtype=torch.bfloat16)
        lse = torch.full((wl.batch, wl.H_qo), float("nan"), device=cuda_device)
        layers.append((inp, o, lse))
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                           max_batch=wl.batch, max_total_qo_rows=wl.batch, num_ctas=148, tile_q=16, pdl=True,
                           max_qo_len=1)
    eng = bsra.Engine(cfg, 0)
    s = torch.cuda.Stream()
    i0 = layers[0][0]

    def step():
        for inp, o, lse in layers:
            eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse,
                    stream=s)

    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        eng.plan(i0.qo_indptr, i0.kv_page_indptr, i0.kv_last_page_len, i0.sm_scale, stream=s)
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    for _, o, lse in layers:
        o.fill_(float("nan"))
        lse.fill_(float("nan"))
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        eng.plan(i0.qo_indptr, i0.kv_page_indptr, i0.kv_last_page_len, i0.sm_scale, stream=s)  # as bench
        g.replay()
        g.replay()
    torch.cuda.synchronize()
    for r in (1, 3):
        inp, o, lse = layers[r]
        assert_close((o.float().cpu().numpy(), lse.cpu().numpy()), oracle.attention_from_inputs(inp), "bf16",
                     what=f"headline graph layer {r}")
    # every layer equals its own eager run bit for bit (graph + PDL change nothing)
    for r in (0, 2):
        inp, o, lse = layers[r]
        o2, l2 = torch.empty_like(o), torch.empty_like(lse)
        eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o2, l2)
        torch.cuda.synchronize()
        assert torch.equal(o2, o) and torch.equal(l2, lse), f"layer {r}: graph replay != eager run"


@pytest.mark.parametrize("S,P", [(4096, 64), (32768, 512)])
def test_quest_block_sparse_decode(cuda_device, S, P):
    """Quest workload: 32 single-head rows, each over `P` scattered pages of a
    32 x S/16-page pool, through the decode kernel as the bench runs it; sampled rows vs oracle."""
    wl, extra = synth.quest_decode(S, P)
    inp = synth.make_inputs(wl, device=cuda_device, extra_pages=extra)
    cfg = bsra.make_config(H_qo=1, H_kv=1, D=128, page_size=16, dtype="bf16", max_batch=wl.batch,
                           max_total_qo_rows=wl.batch, num_ctas=148, tile_q=16, max_qo_len=1)
    eng = bsra.Engine(cfg, 0)
    o = torch.full((wl.batch, 1, 128), float("nan"), device=cuda_device, dtype=torch.bfloat16)
    lse = torch.full((wl.batch, 1), float("nan"), device=cuda_device)
    eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
    eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse)
    torch.cuda.synchronize()
    assert eng.selected_kernel() == "tc_decode"
    reqs = [0, 13, 31]
    ref = oracle.attention_from_inputs(synth.request_subset(inp, reqs))
    assert_close((o[reqs].float().cpu().numpy(), lse[reqs].cpu().numpy()), ref, "bf16", what=f"quest {S}/{P}")
