"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle, element by
element, on the same seeded inputs. Tolerances: BASELINE north_star (1e-2 on o, 1e-3 on lse
for bf16/f16 with fp32 accumulation); fp32 inputs 1e-5."""
import numpy as np
import pytest
import torch

import oracle
import paper_2501_01005_b200 as bsra
import synth
from oracle import scheduler_ref as S
from tests.helpers import assert_close, engine_for, rows_of_requests, run_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("num_ctas", [1, 4, 148, 296])
@pytest.mark.parametrize("permute", [False, True])
def test_c1_tiny_decode_fp32(cuda_device, num_ctas, permute):
    inp = synth.make_inputs(synth.c1_tiny_decode(), device=cuda_device, permute=permute)
    gpu = run_gpu(inp, num_ctas=num_ctas)
    assert_close(gpu, oracle.attention_from_inputs(inp), "f32", what=f"c1 nc={num_ctas}")


def test_c1_plan_device_readback_matches_python(cuda_device):
    inp = synth.make_inputs(synth.c1_tiny_decode(), device=cuda_device)
    _, _, eng = run_gpu(inp, num_ctas=4)
    dev_img = eng.export_plan(from_device=True)
    wl = inp.wl
    ref = S.plan_ref(wl.qo_lens, wl.kv_lens, g=wl.g, H_kv=wl.H_kv, num_ctas=4, align=wl.page_size,
                     qo_begin=inp.qo_indptr[:-1], page_begin=inp.kv_page_indptr[:-1])
    assert np.array_equal(dev_img, ref.image)


@pytest.mark.parametrize("seed", range(36))
def test_random_small_workloads(cuda_device, seed):
    rng = np.random.default_rng(7000 + seed)
    dtype = ["bf16", "f16", "f32"][seed % 3]
    wl = synth.random_workload(rng, dtype=dtype, max_batch=5, max_qo=70, max_kv=300)
    inp = synth.make_inputs(wl, device=cuda_device, seed_base=seed, layout="NHD" if seed % 4 else "HND")
    nc = [1, 3, 16, 148][seed % 4]
    gpu = run_gpu(inp, num_ctas=nc)
    assert_close(gpu, oracle.attention_from_inputs(inp), dtype, what=f"seed {seed} {wl}")


@pytest.mark.parametrize("kernel", ["simt", "auto"])
@pytest.mark.parametrize("mask", ["none", "causal", "custom"])
@pytest.mark.parametrize("tile_q", [16, 64, 128, 256])
def test_tiles_masks_kernels_bf16(cuda_device, kernel, mask, tile_q):
    wl = synth.Workload("t", 32, 8, 128, 16, "bf16", mask, np.array([1, 37, 5, 130, 0], np.int32),
                        np.array([300, 37, 900, 250, 33], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device, seed_base=3)
    gpu = run_gpu(inp, num_ctas=148, tile_q=tile_q, kernel=kernel)
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what=f"{kernel} {mask} T_q={tile_q}")


def test_peaked_logits_bf16(cuda_device):
    wl = synth.Workload("peak", 32, 8, 128, 16, "bf16", "causal", np.array([3, 64], np.int32),
                        np.array([700, 64], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device, q_scale=8.0)
    assert_close(run_gpu(inp, num_ctas=64), oracle.attention_from_inputs(inp), "bf16", what="peaked")


def test_o_fp32_state_output(cuda_device):
    wl = synth.Workload("st", 8, 2, 64, 4, "bf16", "none", np.ones(3, np.int32), np.array([10, 0, 77], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = run_gpu(inp, num_ctas=8, o_dtype="f32")
    assert_close(gpu, oracle.attention_from_inputs(inp), "bf16", what="o f32")


def test_determinism_bitwise(cuda_device):
    wl = synth.c2_decode_llama8b(batch=16)
    inp = synth.make_inputs(wl, device=cuda_device)
    eng = engine_for(wl, num_ctas=296)
    a = run_gpu(inp, eng)
    b = run_gpu(inp, eng)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_num_ctas_agree(cuda_device):
    wl = synth.c2_decode_llama8b(batch=8)
    inp = synth.make_inputs(wl, device=cuda_device)
    ref = oracle.attention_from_inputs(inp)
    for nc in (1, 4, 148, 296):
        assert_close(run_gpu(inp, num_ctas=nc), ref, "bf16", what=f"nc {nc}")


def test_page_size_invariance(cuda_device):
    """Same logical KV in page sizes 1, 4, 16 (independent pools) all match the oracle."""
    for ps in (1, 4, 16):
        wl = synth.Workload("ps", 32, 8, 128, ps, "bf16", "none", np.ones(4, np.int32),
                            np.array([17, 100, 3, 64], np.int32))
        inp = synth.make_inputs(wl, device=cuda_device)
        assert_close(run_gpu(inp, num_ctas=37), oracle.attention_from_inputs(inp), "bf16", what=f"ps {ps}")


def test_graph_capture_and_replan(cuda_device):
    """run() captured once in a CUDA graph; re-plan with new lengths (fixed workspace offsets,
    App. D.1) and replay: outputs follow the new plan."""
    wl1 = synth.Workload("g", 32, 8, 128, 16, "bf16", "none", np.ones(6, np.int32),
                         np.array([100, 200, 300, 400, 500, 600], np.int32))
    wl2 = synth.Workload("g", 32, 8, 128, 16, "bf16", "none", np.ones(6, np.int32),
                         np.array([101, 201, 301, 401, 501, 601], np.int32))
    inp1 = synth.make_inputs(wl1, device=cuda_device, extra_pages=64)
    eng = engine_for(wl1, num_ctas=148, max_batch=8, max_rows=8)
    o = torch.zeros((6, 32, 128), device=cuda_device, dtype=torch.bfloat16)
    lse = torch.zeros((6, 32), device=cuda_device)
    eng.plan(inp1.qo_indptr, inp1.kv_page_indptr, inp1.kv_last_page_len, inp1.sm_scale)
    idx = torch.zeros(4096, dtype=torch.int32, device=cuda_device)
    idx[:inp1.kv_page_indices.numel()] = inp1.kv_page_indices
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        eng.run(inp1.q, inp1.k_pool, inp1.v_pool, inp1.k_strides, inp1.v_strides, idx, o, lse, stream=s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        eng.run(inp1.q, inp1.k_pool, inp1.v_pool, inp1.k_strides, inp1.v_strides, idx, o, lse, stream=s)
    graph.replay()
    torch.cuda.synchronize()
    assert_close((o.float().cpu().numpy(), lse.cpu().numpy()), oracle.attention_from_inputs(inp1), "bf16",
                 what="graph step 1")
    # step 2: one more token per request, pages re-laid out in the same pool
    inp2 = synth.make_inputs(wl2, device=cuda_device, extra_pages=inp1.k_pool.shape[0] - 135)
    inp2.k_pool = inp1.k_pool
    inp2.v_pool = inp1.v_pool
    n2 = inp2.kv_page_indices.numel()
    assert n2 == 135 and inp1.k_pool.shape[0] >= int(inp2.kv_page_indices.max()) + 1
    idx[:n2] = inp2.kv_page_indices
    eng.plan(inp2.qo_indptr, inp2.kv_page_indptr, inp2.kv_last_page_len, inp2.sm_scale, stream=s)
    torch.cuda.synchronize()
    q_dst = inp1.q  # the graph captured inp1.q's address
    q_dst.copy_(inp2.q)
    graph.replay()
    torch.cuda.synchronize()
    inp2.q = q_dst
    inp2.kv_page_indices = idx[:n2]
    assert_close((o.float().cpu().numpy(), lse.cpu().numpy()), oracle.attention_from_inputs(inp2), "bf16",
                 what="graph step 2")


class _GraphRig:
    """Fixed-address buffers sized by engine bounds (q / o / lse rows = max_total_qo_rows, pools,
    page table), so one captured graph can be replayed over a sequence of plans: each workload's
    inputs are copied into the captured addresses before its replay."""

    def __init__(self, dev, H_qo, H_kv, D, ps, max_rows, max_pages):
        self.dev = dev
        self.q = torch.zeros((max_rows, H_qo, D), device=dev, dtype=torch.bfloat16)
        self.o = torch.zeros((max_rows, H_qo, D), device=dev, dtype=torch.bfloat16)
        self.lse = torch.zeros((max_rows, H_qo), device=dev)
        self.k = torch.zeros((max_pages, ps, H_kv, D), device=dev, dtype=torch.bfloat16)
        self.v = torch.zeros_like(self.k)
        self.idx = torch.zeros(max_pages, dtype=torch.int32, device=dev)
        self.s = torch.cuda.Stream()
        self.graph = None

    def load(self, inp):
        nq, npg, nnz = inp.q.shape[0], inp.k_pool.shape[0], inp.kv_page_indices.numel()
        self.q[:nq].copy_(inp.q)
        self.k[:npg].copy_(inp.k_pool)
        self.v[:npg].copy_(inp.v_pool)
        self.idx[:nnz].copy_(inp.kv_page_indices)
        torch.cuda.synchronize()
        return nq

    def run(self, eng):
        eng.run(self.q, self.k, self.v, self.k.stride()[:3], self.v.stride()[:3], self.idx, self.o, self.lse,
                stream=self.s)

    def capture(self, eng):
        with torch.cuda.stream(self.s):
            self.run(eng)  # warm (first-launch attribute setup stays outside the graph)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.s):
            self.run(eng)

    def check(self, inp, nq, what):
        self.o[:nq].fill_(float("nan"))
        torch.cuda.synchronize()
        self.graph.replay()
        torch.cuda.synchronize()
        assert_close((self.o[:nq].float().cpu().numpy(), self.lse[:nq].cpu().numpy()),
                     oracle.attention_from_inputs(inp), "bf16", what=what)


def _dec_wl(qo, kv):
    return synth.Workload("gr", 32, 8, 128, 16, "bf16", "causal", np.array(qo, np.int32), np.array(kv, np.int32))


def test_graph_replay_across_growing_plans(cuda_device):
    """a graph captured once must stay correct when later plans within the
    engine bounds grow the batch, the rows, and l_qo per request. With max_qo_len set, the decode
    kernel's live columns come from the bound, and under capture the q map spans max_total_qo_rows
    rows, so every replay below is of the SAME graph."""
    seq = [_dec_wl([1] * 4, [40, 300, 17, 900]),
           _dec_wl([1, 2, 1, 2, 2, 1, 1, 2], [5, 64, 700, 33, 1200, 16, 2, 257]),
           _dec_wl([2, 2, 2], [3000, 2, 129])]
    rig = _GraphRig(cuda_device, 32, 8, 128, 16, max_rows=16, max_pages=512)
    cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", mask="causal", max_batch=8,
                           max_total_qo_rows=16, max_qo_len=2, num_ctas=148, tile_q=16, pdl=True)
    eng = bsra.Engine(cfg, 0)
    for k, wl in enumerate(seq):
        inp = synth.make_inputs(wl, device=cuda_device, seed_base=10 * k)
        nq = rig.load(inp)
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale, stream=rig.s)
        if rig.graph is None:
            rig.capture(eng)
        rig.check(inp, nq, f"replay {k}")
    with pytest.raises(bsra.BsraError, match="max_qo_len"):
        inp = synth.make_inputs(_dec_wl([3], [50]), device=cuda_device)
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)


def test_graph_guard_rejects_replans_a_replay_cannot_run(cuda_device):
    """Without max_qo_len the live columns follow the plan. After a capture at l_qo = 1 (4 live
    columns), a plan needing 8 columns, or another query tile, fails with EBOUNDS and keeps the
    old plan (the graph still replays it correctly); bsra_graph_release lifts the guard and a
    re-captured graph runs the new plan."""
    rig = _GraphRig(cuda_device, 32, 8, 128, 16, max_rows=64, max_pages=512)
    cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", mask="causal", max_batch=8,
                           max_total_qo_rows=64, num_ctas=148, tile_set=(16, 64, 128))
    eng = bsra.Engine(cfg, 0)
    wl1 = _dec_wl([1] * 5, [40, 300, 17, 900, 64])
    inp1 = synth.make_inputs(wl1, device=cuda_device)
    nq1 = rig.load(inp1)
    eng.plan(inp1.qo_indptr, inp1.kv_page_indptr, inp1.kv_last_page_len, inp1.sm_scale, stream=rig.s)
    rig.capture(eng)
    rig.check(inp1, nq1, "captured plan")
    grow_cols = synth.make_inputs(_dec_wl([1, 2, 1], [40, 300, 17]), device=cuda_device, seed_base=1)
    grow_tile = synth.make_inputs(_dec_wl([40, 1], [40, 300]), device=cuda_device, seed_base=2)
    for inp, why in ((grow_cols, "live columns"), (grow_tile, "query tile")):
        with pytest.raises(bsra.BsraError, match=why):
            eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale, stream=rig.s)
        rig.check(inp1, nq1, f"old plan kept after a refused re-plan ({why})")
    # shrinking within the captured choices is fine without a release
    inp3 = synth.make_inputs(_dec_wl([1] * 3, [5, 6, 700]), device=cuda_device, seed_base=3)
    nq3 = rig.load(inp3)
    eng.plan(inp3.qo_indptr, inp3.kv_page_indptr, inp3.kv_last_page_len, inp3.sm_scale, stream=rig.s)
    rig.check(inp3, nq3, "smaller plan, same graph")
    eng.graph_release()
    nq = rig.load(grow_cols)
    eng.plan(grow_cols.qo_indptr, grow_cols.kv_page_indptr, grow_cols.kv_last_page_len, grow_cols.sm_scale,
             stream=rig.s)
    rig.capture(eng)
    rig.check(grow_cols, nq, "re-captured after release")


def test_bounds_are_enforced(cuda_device):
    wl = synth.Workload("b", 8, 2, 64, 4, "bf16", "none", np.ones(3, np.int32), np.array([5, 6, 7], np.int32))
    eng = engine_for(wl, max_batch=2, max_rows=2)
    inp = synth.make_inputs(wl, device=cuda_device)
    with pytest.raises(bsra.BsraError, match="max_batch"):
        eng.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len)


# ------------------------------------------------------------------------ ⊕ kernels
@pytest.mark.parametrize("D", [64, 128])
@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_merge_states_matches_oracle(cuda_device, D, dt):
    g = torch.Generator(device="cpu").manual_seed(5)
    rows, heads = 37, 8
    oa = (torch.rand((rows, heads, D), generator=g) * 2 - 1).to(dt)
    ob = (torch.rand((rows, heads, D), generator=g) * 2 - 1).to(dt)
    la = torch.randn((rows, heads), generator=g) * 4
    lb = torch.randn((rows, heads), generator=g) * 4
    la[0, :] = -float("inf")
    lb[1, :] = -float("inf")
    la[2, :] = -float("inf")
    lb[2, :] = -float("inf")
    oa[2] = 0
    ob[2] = 0
    o, l = bsra.merge_states(oa.to(cuda_device), la.to(cuda_device), ob.to(cuda_device), lb.to(cuda_device),
                             o_out=torch.empty((rows, heads, D), device=cuda_device, dtype=torch.float32))
    ro, rl = oracle.merge(oa.double().numpy(), la.double().numpy(), ob.double().numpy(), lb.double().numpy())
    assert np.max(np.abs(o.cpu().numpy() - ro)) < 1e-5
    fin = np.isfinite(rl)
    assert np.array_equal(np.isneginf(l.cpu().numpy()), ~fin)
    assert np.max(np.abs(l.cpu().numpy()[fin] - rl[fin])) < 1e-5


def test_merge_many_matches_oracle(cuda_device):
    g = torch.Generator(device="cpu").manual_seed(6)
    P, rows, heads, D = 5, 11, 4, 128
    op = torch.rand((P, rows, heads, D), generator=g) * 2 - 1
    lp = torch.randn((P, rows, heads), generator=g) * 3
    lp[2, 3] = -float("inf")
    o = torch.empty((rows, heads, D), device=cuda_device)
    l = torch.empty((rows, heads), device=cuda_device)
    bsra.merge_many(op.to(cuda_device), lp.to(cuda_device), o, l)
    ro, rl = oracle.merge_all([(op[i].double().numpy(), lp[i].double().numpy()) for i in range(P)])
    assert np.max(np.abs(o.cpu().numpy() - ro)) < 1e-5
    assert np.max(np.abs(l.cpu().numpy() - rl)) < 1e-5


# ------------------------------------------------------------- full BASELINE sizes
def test_c2_full_size_sampled(cuda_device):
    """configs[1] at full size in the bench's launch configuration (num_ctas 296); sampled
    requests (short, median, long) compared element by element with the oracle."""
    wl = synth.c2_decode_llama8b()
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = run_gpu(inp, num_ctas=296, tile_q=16)
    order = np.argsort(wl.kv_lens)
    reqs = sorted({int(order[0]), int(order[len(order) // 2]), int(order[-1]), 0, 77})
    ref = oracle.attention_from_inputs(inp, req_list=reqs)
    assert_close(gpu, ref, "bf16", rows=rows_of_requests(inp, reqs), what="c2 sampled")


def test_c3_full_size_sampled(cuda_device):
    """configs[2] (ragged causal prefill, 64/8 heads) at full size; the shortest and one long
    request checked element by element."""
    wl = synth.c3_prefill_llama70b()
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = run_gpu(inp, num_ctas=148)
    order = np.argsort(wl.qo_lens)
    reqs = sorted({int(order[0]), int(order[3])})
    ref = oracle.attention_from_inputs(inp, req_list=reqs)
    assert_close(gpu, ref, "bf16", rows=rows_of_requests(inp, reqs), what="c3 sampled")
