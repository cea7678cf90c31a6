"""Device-side Algorithm 1 (bsra_plan_device; the paper's future work): the plan image the
device kernel builds equals the host scheduler's bit for bit (which tests/test_abi_host.py ties to
oracle/scheduler_ref.py and tests/test_alg1_order.py to the hand traces), on random workloads and
the BASELINE shapes; attention run on a device-built plan matches the oracle; a CUDA graph that
captures plan_device + run replays correctly as the device-side lengths change between steps;
malformed arrays give an empty plan and a status code."""
import numpy as np
import pytest
import torch

import oracle
import paper_2501_01005_b200 as bsra
import synth
from tests.helpers import assert_close

pytestmark = pytest.mark.gpu

MASKS = ["none", "causal", "custom"]


def _bsr(qo, kv, ps):
    qo = np.asarray(qo, np.int64)
    kv = np.asarray(kv, np.int64)
    n = (kv + ps - 1) // ps
    qi = np.concatenate([[0], np.cumsum(qo)]).astype(np.int32)
    ki = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    last = np.where(n > 0, kv - (n - 1) * ps, 0).astype(np.int32)
    return qi, ki, last


def _compare(dev, qo, kv, *, H_qo, H_kv, ps, mask, nc, tile_q, window=0, align=0, L_min=0, alpha=1, beta=1):
    qi, ki, last = _bsr(qo, kv, ps)
    B = len(qo)
    cfg = bsra.make_config(H_qo=H_qo, H_kv=H_kv, D=128, page_size=ps, dtype="bf16", mask=mask, max_batch=max(1, B),
                           max_total_qo_rows=max(1, int(np.sum(qo))), num_ctas=nc, tile_q=tile_q, window=window,
                           kv_chunk_align=align, kv_chunk_min=L_min, alpha=alpha, beta=beta,
                           max_qo_len=max(1, int(np.max(qo, initial=1))))
    host = bsra.plan_host(cfg, nc, qi, ki, last)
    eng = bsra.Engine(cfg, 0)
    t = lambda a: torch.from_numpy(a).to(dev)
    eng.plan_device(B, t(qi), t(ki), t(last))
    assert eng.plan_device_status() == 0
    img = eng.export_plan(from_device=True)
    assert np.array_equal(img, host), (len(img), len(host))
    return img


@pytest.mark.parametrize("seed", range(120))
def test_device_plan_bit_exact(cuda_device, seed):
    rng = np.random.default_rng(77000 + seed)
    B = int(rng.integers(1, 40))
    H_kv = int(rng.choice([1, 2, 8]))
    g = int(rng.choice([1, 4, 8]))
    mask = int(rng.integers(0, 3))
    ps = int(rng.choice([1, 4, 16]))
    tile_q = int(rng.choice([16, 64, 128, 256]))
    qo = rng.integers(0, 3, B) if tile_q == 16 else rng.integers(0, 200, B)
    kv = rng.integers(0, 5000, B) if seed % 3 else np.minimum(rng.zipf(1.3, B) * 50, 150000)
    if mask == 1:
        kv = np.maximum(kv, qo)
    nc = int(rng.choice([1, 7, 148, 296]))
    window = int(rng.choice([0, 0, 64, 1000]))
    _compare(cuda_device, qo, kv, H_qo=H_kv * g, H_kv=H_kv, ps=ps, mask=MASKS[mask], nc=nc, tile_q=tile_q,
             window=window, align=int(rng.choice([0, 1, 32])), L_min=int(rng.choice([0, 500])),
             alpha=int(rng.choice([1, 3])), beta=int(rng.choice([1, 2])))


def test_device_plan_bit_exact_baseline_shapes(cuda_device):
    c2 = synth.c2_decode_llama8b()
    _compare(cuda_device, c2.qo_lens, c2.kv_lens, H_qo=32, H_kv=8, ps=16, mask="none", nc=148, tile_q=16)
    c3 = synth.c3_prefill_llama70b()
    _compare(cuda_device, c3.qo_lens, c3.kv_lens, H_qo=64, H_kv=8, ps=16, mask="causal", nc=148, tile_q=256)
    c5 = synth.c5_long_decode()
    img = _compare(cuda_device, c5.qo_lens, c5.kv_lens, H_qo=32, H_kv=8, ps=16, mask="none", nc=148, tile_q=16)
    assert img[7] > 0  # split rows and merge lists exercised


def test_device_plan_runs_and_graph_replays_new_lengths(cuda_device):
    """One graph = {plan_device from device arrays, run}; between replays only the device-side
    lengths / page table change (no host planning): every replay matches the oracle."""
    max_b, max_pages = 8, 600
    cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", mask="causal", max_batch=max_b,
                           max_total_qo_rows=16, max_qo_len=2, num_ctas=148, tile_q=16, pdl=True)
    eng = bsra.Engine(cfg, 0)
    q = torch.zeros((16, 32, 128), device=cuda_device, dtype=torch.bfloat16)
    kp = torch.zeros((max_pages, 16, 8, 128), device=cuda_device, dtype=torch.bfloat16)
    vp = torch.zeros_like(kp)
    o = torch.zeros((16, 32, 128), device=cuda_device, dtype=torch.bfloat16)
    lse = torch.zeros((16, 32), device=cuda_device)
    d_qi = torch.zeros(max_b + 1, dtype=torch.int32, device=cuda_device)
    d_ki = torch.zeros(max_b + 1, dtype=torch.int32, device=cuda_device)
    d_last = torch.zeros(max_b, dtype=torch.int32, device=cuda_device)
    d_idx = torch.zeros(max_pages, dtype=torch.int32, device=cuda_device)
    s = torch.cuda.Stream()
    B = 6  # fixed batch per captured graph; lengths vary
    steps = [([1, 2, 1, 1, 2, 1], [40, 700, 17, 1, 3000, 255]), ([2, 2, 1, 1, 1, 1], [41, 701, 18, 2, 3001, 256]),
             ([1, 1, 1, 2, 1, 1], [5000, 3, 129, 64, 1, 900])]
    g = None
    for k, (qo, kv) in enumerate(steps):
        wl = synth.Workload("dp", 32, 8, 128, 16, "bf16", "causal", np.array(qo, np.int32), np.array(kv, np.int32))
        inp = synth.make_inputs(wl, device=cuda_device, seed_base=k)
        nq, npg = inp.q.shape[0], inp.k_pool.shape[0]
        q[:nq].copy_(inp.q)
        kp[:npg].copy_(inp.k_pool)
        vp[:npg].copy_(inp.v_pool)
        d_idx[:inp.kv_page_indices.numel()].copy_(inp.kv_page_indices)
        d_qi[:B + 1].copy_(torch.from_numpy(inp.qo_indptr))
        d_ki[:B + 1].copy_(torch.from_numpy(inp.kv_page_indptr))
        d_last[:B].copy_(torch.from_numpy(inp.kv_last_page_len))
        torch.cuda.synchronize()

        def step():
            eng.plan_device(B, d_qi, d_ki, d_last, inp.sm_scale, stream=s)
            eng.run(q, kp, vp, kp.stride()[:3], vp.stride()[:3], d_idx, o, lse, stream=s)
        if g is None:
            with torch.cuda.stream(s):
                step()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                step()
        o.fill_(float("nan"))
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        assert eng.plan_device_status(stream=s) == 0
        assert_close((o[:nq].float().cpu().numpy(), lse[:nq].cpu().numpy()), oracle.attention_from_inputs(inp),
                     "bf16", what=f"device plan step {k}")


def test_device_plan_reports_malformed_arrays(cuda_device):
    cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", max_batch=4, max_total_qo_rows=4,
                           max_qo_len=1, num_ctas=16, tile_q=16)
    eng = bsra.Engine(cfg, 0)
    t = lambda a: torch.tensor(a, dtype=torch.int32, device=cuda_device)
    eng.plan_device(2, t([0, 1, 2]), t([0, 3, 2]), t([16, 1]))  # kv_page_indptr decreasing
    assert eng.plan_device_status() == 1
    assert eng.export_plan(from_device=True)[5] == 0  # empty plan
    eng.plan_device(2, t([0, 1, 2]), t([0, 3, 5]), t([17, 1]))  # last_page_len > page_size
    assert eng.plan_device_status() == 1
    eng.plan_device(2, t([0, 1, 2]), t([0, 3, 5]), t([16, 1]))
    assert eng.plan_device_status() == 0


def test_device_plan_requirements():
    cfg = bsra.make_config(H_qo=32, H_kv=8, D=128, page_size=16, dtype="bf16", max_batch=4, max_total_qo_rows=4,
                           num_ctas=16)  # no fixed tile
    eng = bsra.Engine(cfg, 0)
    z = torch.zeros(8, dtype=torch.int32, device="cuda:0")
    with pytest.raises(bsra.BsraError, match="tile_q"):
        eng.plan_device(2, z, z, z)
