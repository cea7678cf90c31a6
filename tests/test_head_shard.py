"""KV-head sharding (BASELINE north_star "requests and KV heads sharded with
no communication") and the host-side partition functions of the C ABI (include/bsra_dist.h).

CPU: bsra_dist_head_shard / bsra_dist_shard_bsr against their definitions; the oracle's head
shards concatenate to the whole output bit for bit (attention is per head); a world-size-2
gloo group in which every rank takes its head range from libbsra, computes its shard and
all-gathers. GPU: simulated ranks on one device, each with its own engine over H_kv/P heads and
pools holding only those heads, at the configs[1] and configs[2] shapes, against the oracle."""
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
from tests.helpers import assert_close, engine_for, rows_of_requests, run_gpu


@pytest.mark.parametrize("H_kv", [1, 2, 3, 8, 64])
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_head_shard_partition(H_kv, P):
    rng = [bsra.head_shard(H_kv, P, r) for r in range(P)]
    assert rng[0][0] == 0 and rng[-1][1] == H_kv
    for (a, b), (c, d) in zip(rng, rng[1:]):
        assert b == c
    sizes = [b - a for a, b in rng]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 0


def test_head_shard_rejects_bad_arguments():
    for args in ((0, 1, 0), (8, 0, 0), (8, 2, 2), (8, 2, -1)):
        with pytest.raises(bsra.BsraError):
            bsra.head_shard(*args)


def _table(rng, B, ps):
    n = rng.integers(0, 40, B)
    n[rng.random(B) < 0.2] = 0
    n[0] = 1  # fewer pages than ranks
    indptr = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    idx = rng.permutation(int(indptr[-1]) + 7)[:int(indptr[-1])].astype(np.int32)
    last = np.where(n > 0, rng.integers(1, ps + 1, B), 0).astype(np.int32)
    return indptr, idx, last


@pytest.mark.parametrize("seed", range(40))
def test_shard_bsr_matches_definition(seed):
    """bsra_dist_shard_bsr against its definition written out here: rank r keeps logical pages
    [floor(r n / P), floor((r+1) n / P)) of each request; the request's last_page_len only on the
    rank holding its final page; shard lengths add up to the request's l_kv."""
    rng = np.random.default_rng(seed)
    ps = int(rng.choice([1, 4, 16]))
    B = int(rng.integers(1, 9))
    indptr, idx, last = _table(rng, B, ps)
    P = int(rng.choice([1, 2, 3, 8]))
    total = np.zeros(B, np.int64)
    for r in range(P):
        ip, ix, lp = bsra.sequence_shard(indptr, idx, last, ps, P, r)
        want_ip, want_ix, want_lp = [0], [], []
        for i in range(B):
            n = int(indptr[i + 1] - indptr[i])
            a, b = r * n // P, (r + 1) * n // P
            want_ix += list(idx[indptr[i] + a:indptr[i] + b])
            want_ip.append(len(want_ix))
            want_lp.append(int(last[i]) if (b == n and b > a) else ps)
        assert ip.tolist() == want_ip and ix.tolist() == want_ix and lp.tolist() == want_lp
        n_r = ip[1:] - ip[:-1]
        total += np.where(n_r > 0, (n_r - 1) * ps + lp, 0)
    n = indptr[1:] - indptr[:-1]
    assert np.array_equal(total, np.where(n > 0, (n - 1) * ps + last, 0))


def test_shard_bsr_rejects_malformed_tables():
    ip = np.array([0, 2, 3], np.int32)
    idx = np.arange(3, dtype=np.int32)
    with pytest.raises(bsra.BsraError):
        bsra.sequence_shard(ip, idx, np.array([0, 1], np.int32), 4, 2, 0)  # last_page_len 0 with pages
    with pytest.raises(bsra.BsraError):
        bsra.sequence_shard(ip, idx, np.array([5, 1], np.int32), 4, 2, 0)  # > page_size
    with pytest.raises(bsra.BsraError):
        bsra.sequence_shard(ip, idx, np.array([1, 1], np.int32), 4, 2, 2)  # rank out of range
    with pytest.raises(bsra.BsraError):
        bsra.sequence_shard(np.array([0, 2, 1], np.int32), idx, np.array([1, 1], np.int32), 4, 2, 0)


def _oracle_heads(inp, h0, h1):
    return oracle.attention_from_inputs(synth.head_slice(inp, h0, h1))


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("mask", ["none", "causal"])
def test_oracle_head_shards_concatenate_to_whole(P, mask):
    """Attention is computed per (kv head, qo head group): the head shards of the oracle,
    concatenated along heads, ARE the whole output — no collective is needed."""
    wl = synth.Workload("hs", 32, 8, 32, 4, "bf16", mask, np.array([1, 3, 2], np.int32),
                        np.array([9, 40, 2], np.int32))
    inp = synth.make_inputs(wl)
    whole = oracle.attention_from_inputs(inp)
    parts = [_oracle_heads(inp, *bsra.head_shard(wl.H_kv, P, r)) for r in range(P)]
    o = np.concatenate([p[0] for p in parts], axis=1)
    l = np.concatenate([p[1] for p in parts], axis=1)
    assert np.array_equal(o, whole[0]) and np.array_equal(l, whole[1])


def _gloo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = synth.Workload("hs", 16, 4, 32, 4, "bf16", "causal", np.array([2, 1, 5], np.int32),
                            np.array([7, 33, 5], np.int32))
        inp = synth.make_inputs(wl)
        h0, h1 = bsra.head_shard(wl.H_kv, world, rank)  # the rank's heads, from libbsra
        o, l = _oracle_heads(inp, h0, h1)
        og = [torch.empty_like(torch.from_numpy(o)) for _ in range(world)]
        lg = [torch.empty_like(torch.from_numpy(l)) for _ in range(world)]
        dist.all_gather(og, torch.from_numpy(o))  # only to compare here: the method needs none
        dist.all_gather(lg, torch.from_numpy(l))
        whole = oracle.attention_from_inputs(inp)
        ok = np.array_equal(torch.cat(og, 1).numpy(), whole[0]) and np.array_equal(torch.cat(lg, 1).numpy(), whole[1])
        q.put((rank, (h0, h1), ok))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_head_shards():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [(0, 2), (2, 4)]
    assert all(r[2] for r in res)


# --------------------------------------------------------------------------------- GPU
def _gpu_head_sharded(inp, P, **kw):
    """Simulated ranks on one GPU: per rank an engine over its kv heads and pools holding only
    those heads (what each GPU of a P-way head-sharded run holds); outputs concatenated."""
    os_, ls_ = [], []
    for r in range(P):
        h0, h1 = bsra.head_shard(inp.wl.H_kv, P, r)
        part = synth.head_slice(inp, h0, h1)
        o, l, eng = run_gpu(part, **kw)
        os_.append(o)
        ls_.append(l)
        del part, eng
    return np.concatenate(os_, axis=1), np.concatenate(ls_, axis=1)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 8])
def test_c2_head_sharded_full_size(cuda_device, P):
    """configs[1] (batch 128, 32/8 heads, ShareGPT-like lengths) split over P ranks by kv head, in
    the bench's launch configuration (148 CTAs, T_q 16); sampled requests vs the oracle."""
    inp = synth.make_inputs(synth.c2_decode_llama8b(), device=cuda_device)
    gpu = _gpu_head_sharded(inp, P, num_ctas=148, tile_q=16)
    order = np.argsort(inp.wl.kv_lens)
    reqs = sorted({int(order[0]), int(order[64]), int(order[-1])})
    assert_close(gpu, oracle.attention_from_inputs(inp, req_list=reqs), "bf16",
                 rows=rows_of_requests(inp, reqs), what=f"c2 head-sharded P={P}")


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 8])
def test_c3_head_sharded_sampled(cuda_device, P):
    """configs[2] (causal prefill, 64/8 heads) split by kv head; per-rank plans differ (fewer
    rows => different L), so equality with the oracle is within tolerance, not bitwise."""
    wl = synth.c3_prefill_llama70b()
    inp = synth.make_inputs(wl, device=cuda_device)
    gpu = _gpu_head_sharded(inp, P, num_ctas=148)
    order = np.argsort(wl.qo_lens)
    reqs = [int(order[0]), int(order[2])]
    assert_close(gpu, oracle.attention_from_inputs(inp, req_list=reqs), "bf16",
                 rows=rows_of_requests(inp, reqs), what=f"c3 head-sharded P={P}")


@pytest.mark.gpu
def test_small_head_sharded_all_rows(cuda_device):
    wl = synth.Workload("hs", 32, 8, 128, 16, "bf16", "causal", np.array([1, 3, 1, 40], np.int32),
                        np.array([70, 300, 2, 900], np.int32))
    inp = synth.make_inputs(wl, device=cuda_device)
    whole = oracle.attention_from_inputs(inp)
    for P in (1, 2, 3, 8):
        assert_close(_gpu_head_sharded(inp, P, num_ctas=37), whole, "bf16", what=f"P={P}")


def test_request_subset_is_data_movement_only():
    """synth.request_subset (used to check a few requests of multi-GB workloads) gives the oracle
    exactly the rows of those requests (bitwise)."""
    wl = synth.Workload("x", 8, 2, 32, 4, "bf16", "causal", np.array([2, 1, 3], np.int32),
                        np.array([9, 40, 3], np.int32))
    inp = synth.make_inputs(wl)
    full = oracle.attention_from_inputs(inp)
    sub = oracle.attention_from_inputs(synth.request_subset(inp, [1, 2]))
    rows = rows_of_requests(inp, [1, 2])
    assert np.array_equal(full[0][rows], sub[0]) and np.array_equal(full[1][rows], sub[1])
