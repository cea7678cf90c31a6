"""Long-context sequence split (BASELINE configs[4]): each rank owns a contiguous 1/P of every
request's pages; partial states (o, lse) are gathered and combined with ⊕ in rank order
(PAPER.md:129).  CPU: the page partition and the gather+merge host logic over a real
torch.distributed gloo group (world size 2).  GPU: simulated ranks on one device, and the
library's NCCL path (bsra_dist) on one rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2501_01005_b200 as bsra
import synth
from synth import raw_bits


def _wl(kv=(1, 50, 133, 4000)):
    return synth.Workload("seq", 8, 2, 32, 4, "bf16", "none", np.ones(len(kv), np.int32), np.array(kv, np.int32))


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_sequence_shard_partitions_pages(P):
    inp = synth.make_inputs(_wl())
    idx = inp.kv_page_indices.numpy()
    shards = [bsra.sequence_shard(inp.kv_page_indptr, idx, inp.kv_last_page_len, 4, P, r) for r in range(P)]
    for i in range(inp.wl.batch):
        got = np.concatenate([s[1][s[0][i]:s[0][i + 1]] for s in shards])
        want = idx[inp.kv_page_indptr[i]:inp.kv_page_indptr[i + 1]]
        assert np.array_equal(got, want)
        # only the rank holding the request's final page carries its last_page_len
        lens = [(s[0][i + 1] - s[0][i] - 1) * 4 + s[2][i] if s[0][i + 1] > s[0][i] else 0 for s in shards]
        assert sum(lens) == inp.wl.kv_lens[i]


def _shard_oracle(inp, P, r):
    wl = inp.wl
    ki, kx, kl = bsra.sequence_shard(inp.kv_page_indptr, inp.kv_page_indices.numpy(), inp.kv_last_page_len,
                                     wl.page_size, P, r)
    return oracle.paged_attention(
        qo_indptr=inp.qo_indptr, kv_page_indptr=ki, kv_last_page_len=kl, kv_page_indices=kx, q=raw_bits(inp.q),
        k_pool=raw_bits(inp.k_pool), v_pool=raw_bits(inp.v_pool), k_strides=inp.k_strides, v_strides=inp.v_strides,
        H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, sm_scale=inp.sm_scale)


def _gloo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inp = synth.make_inputs(_wl())
        o, l = _shard_oracle(inp, world, rank)
        ot, lt = torch.from_numpy(o), torch.from_numpy(l)
        og = [torch.empty_like(ot) for _ in range(world)]
        lg = [torch.empty_like(lt) for _ in range(world)]
        dist.all_gather(og, ot)
        dist.all_gather(lg, lt)
        mo, ml = oracle.merge_all([(og[k].numpy(), lg[k].numpy()) for k in range(world)])
        full = oracle.attention_from_inputs(inp)
        q.put((rank, float(np.max(np.abs(mo - full[0]))), float(np.max(np.abs(ml - full[1]))),
               mo.tobytes() == og[0].numpy().tobytes() if world == 1 else None))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_two_rank_gather_merge_equals_whole():
    """world size 2 over gloo: shard -> per-rank state -> all_gather -> ⊕ in rank order == oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, do, dl, _ in res:
        assert do < 1e-12 and dl < 1e-12, (rank, do, dl)


# --------------------------------------------------------------------------------- GPU
def _gpu_shard_states(inp, P, dev, nc=148):
    """Simulated ranks on one GPU: per shard one engine run with fp32 state output."""
    wl = inp.wl
    nq = int(inp.qo_indptr[-1])
    os_, ls_ = [], []
    for r in range(P):
        ki, kx, kl = bsra.sequence_shard(inp.kv_page_indptr, inp.kv_page_indices.cpu().numpy(), inp.kv_last_page_len,
                                         wl.page_size, P, r)
        cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                               o_dtype="f32", max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=nc, tile_q=16)
        eng = bsra.Engine(cfg, 0)
        o = torch.empty((nq, wl.H_qo, wl.D), device=dev)
        l = torch.empty((nq, wl.H_qo), device=dev)
        eng.plan(inp.qo_indptr, ki, kl, inp.sm_scale)
        eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, torch.from_numpy(kx).to(dev), o, l)
        os_.append(o)
        ls_.append(l)
    torch.cuda.synchronize()
    return torch.stack(os_), torch.stack(ls_)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_gpu_simulated_ranks_merge_many(cuda_device, P):
    from tests.helpers import assert_close
    wl = synth.Workload("seq", 32, 8, 128, 16, "bf16", "none", np.ones(3, np.int32),
                        np.array([70000, 9000, 333], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    op, lp = _gpu_shard_states(inp, P, cuda_device)
    o = torch.empty((3, 32, 128), device=cuda_device, dtype=torch.bfloat16)
    l = torch.empty((3, 32), device=cuda_device)
    bsra.merge_many(op, lp, o, l)
    torch.cuda.synchronize()
    assert_close((o.float().cpu().numpy(), l.cpu().numpy()), oracle.attention_from_inputs(inp), "bf16",
                 what=f"simulated P={P}")


@pytest.mark.gpu
def test_gpu_nccl_single_rank_equals_simulated(cuda_device):
    """The library's NCCL all-gather + ⊕ on one rank is bitwise the simulated-rank merge."""
    wl = synth.Workload("seq", 32, 8, 128, 16, "bf16", "none", np.ones(2, np.int32), np.array([5000, 77], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    op, lp = _gpu_shard_states(inp, 1, cuda_device)
    uid = bsra.Dist.unique_id()
    d = bsra.Dist(1, 0, uid, 0)
    scratch = d.scratch(2, 32, 128, cuda_device)
    o1 = torch.empty((2, 32, 128), device=cuda_device, dtype=torch.bfloat16)
    l1 = torch.empty((2, 32), device=cuda_device)
    d.allgather_merge(op[0], lp[0], scratch, o1, l1)
    o2 = torch.empty_like(o1)
    l2 = torch.empty_like(l1)
    bsra.merge_many(op, lp, o2, l2)
    torch.cuda.synchronize()
    d.close()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.gpu
@pytest.mark.parametrize("nc", [148, 37])
def test_balance_ctas_flag(cuda_device, nc):
    """BSRA_FLAG_BALANCE_CTAS: Algorithm 1 with the queue count c <= num_ctas of smallest makespan,
    the grid unchanged (empty queues exit). Few long rows (configs[4]'s shape, shorter): the
    makespan does not grow, and o / lse match the oracle and the unbalanced plan."""
    import paper_2501_01005_b200 as bsra
    from tests.helpers import assert_close, run_gpu
    wl = synth.Workload("long_small", 32, 8, 128, 16, "bf16", "none", np.ones(4, np.int32),
                        np.full(4, 18_500, np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    res = {}
    for bal in (False, True):
        cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                               max_batch=wl.batch, max_total_qo_rows=wl.batch, num_ctas=nc, tile_q=16,
                               balance_ctas=bal)
        eng = bsra.Engine(cfg, 0)
        gpu = run_gpu(inp, eng)
        costs, mk = eng.plan_stats()
        assert len(costs) == nc  # the grid (and a captured graph) keep num_ctas CTAs
        res[bal] = (gpu, mk, int((costs > 0).sum()))
    assert res[True][1] <= res[False][1]
    ref = oracle.attention_from_inputs(inp)
    assert_close(res[True][0], ref, "bf16", what=f"balanced nc={nc}")
    assert np.max(np.abs(res[True][0][0] - res[False][0][0])) < 1e-2
