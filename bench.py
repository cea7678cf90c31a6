#!/usr/bin/env python
"""bench.py — paged decode HBM TB/s (BASELINE.json configs[1]) on B200, plus the prefill
TFLOP/s of configs[2] as a secondary figure, through the libbsra C ABI.

A step = one decode generation step of the hot path for a
Llama-3-8B-shaped model: plan() once (host Algorithm 1 + H2D of the plan image) and
run() for every one of `--layers` layers (distinct q / KV pools / o per layer, the same plan,
replayed from one CUDA graph). value = KV bytes (+ q, o, lse, indices) per step /
device time. Every layer's KV pool is 621 MB >> 126 MB L2, so no layer is L2-resident when
it is read (no flush needed; stated in config).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1: launched under torchrun (or `--gpus N` alone re-launches itself under torchrun), one
rank per GPU. Headline: every rank runs its own configs[1] batch (requests sharded, no
collective on the data path) -> "scaling": "weak"; the time is the max over ranks. Secondary
keys shard the FIXED workload: configs[1] and configs[2] / configs[3] by KV head (no
collective, strong scaling), configs[4] along the sequence (NCCL all-gather + merge).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ["NCCL_DEBUG"] = os.environ.get("BSRA_NCCL_DEBUG", "WARN")
# stdout carries exactly one JSON line. Anything a library prints to the process's stdout (NCCL's
# version banner is printed at WARN level) goes to stderr: fd 1 is pointed at fd 2, and the JSON
# line is written through a duplicate of the original stdout.
_JSON_OUT = os.fdopen(os.dup(1), "w")
sys.stdout.flush()
os.dup2(2, 1)


def emit(obj) -> None:
    _JSON_OUT.write(json.dumps(obj) + "\n")
    _JSON_OUT.flush()

import synth  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# BASELINE.json's metric, printed identically by both arms (the driver pairs them by it)
METRIC = "paged decode HBM TB/s & prefill TFLOP/s (% roofline) at 1/2/4/8 B200"
FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return FALLBACK, "fallback"


# ------------------------------------------------------------------ clocks ---
class ClockSampler:
    """SM clock / throttle-reason sampling (NVML, every 10 ms) during the timed region
    (B200_PROFILING.md clocks line); falls back to nvidia-smi if NVML is unavailable."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake_slowdown": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self.stop_flag = threading.Event()
        self.thread = None
        self.max_mhz = None

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.dev]) if vis else self.dev
            h = N.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            masks = {k: getattr(N, v) for k, v in self.REASONS.items() if hasattr(N, v)}

            def loop():
                while not self.stop_flag.is_set():
                    try:
                        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, [k for k, m in masks.items() if r & m]))
                    except Exception:
                        pass
                    time.sleep(0.01)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None

    def stop(self):
        self.stop_flag.set()
        if self.thread is not None:
            self.thread.join(timeout=1)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        sm = [x[0] for x in self.samples]
        reasons = sorted({k for _, rs in self.samples for k in rs})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "sm_mhz_min": min(sm)}


# --------------------------------------------------------------- workloads ---
def decode_bytes(wl) -> dict:
    """Algorithmic bytes of one decode layer: every KV byte once per kv head,
    plus q, o (dtype), lse (fp32) and the BSR arrays (int32)."""
    es = 2 if wl.dtype in ("bf16", "f16") else 4
    kv_es = 1 if wl.kv_dtype == "e4m3" else es  # fp8 KV cache: one byte per element (NEXT-2)
    kv = int(wl.kv_lens.astype(np.int64).sum()) * wl.H_kv * wl.D * 2 * kv_es
    nq = int(wl.qo_lens.sum())
    qo = 2 * nq * wl.H_qo * wl.D * es + nq * wl.H_qo * 4
    idx = int(wl.num_pages().sum()) * 4 + 3 * (wl.batch + 1) * 4
    return {"kv": kv, "total": kv + qo + idx}


def causal_flops(wl) -> float:
    """4*D flops per visible (query, key, qo head) pair."""
    pairs = 0
    for lq, lk in zip(wl.qo_lens.astype(np.int64), wl.kv_lens.astype(np.int64)):
        # right-aligned causal: row r sees min(lk, lk - lq + r + 1) keys
        r = np.arange(lq)
        pairs += int(np.clip(lk - lq + r + 1, 0, lk).sum())
    return 4.0 * wl.D * wl.H_qo * pairs


class Layered:
    """R layers of one workload: per-layer q / K / V pools / o, one shared page table."""

    def __init__(self, wl, layers, device, seed_base=0):
        import paper_2501_01005_b200 as bsra
        self.wl = wl
        self.layers = []
        for r in range(layers):
            inp = synth.make_inputs(wl, device=device, seed_base=seed_base + 100 * r)
            nq = int(inp.qo_indptr[-1])
            o = torch.empty((nq, wl.H_qo, wl.D), device=device, dtype=inp.q.dtype)
            lse = torch.empty((nq, wl.H_qo), device=device)
            if r > 0:  # one page table per model (shared by all layers)
                inp.kv_page_indices = self.layers[0][0].kv_page_indices
            self.layers.append((inp, o, lse))
        self.inp0 = self.layers[0][0]
        self.bsra = bsra

    def engine(self, **kw):
        wl = self.wl
        if wl.kv_dtype:
            kw = dict(kw, kv_dtype=wl.kv_dtype, k_scale=self.inp0.k_scale, v_scale=self.inp0.v_scale)
        if wl.rope_theta:
            kw = dict(kw, rope_theta=wl.rope_theta, rope_scale=wl.rope_scale)
        cfg = self.bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                                    mask=wl.mask, max_batch=wl.batch, max_total_qo_rows=int(wl.qo_lens.sum()),
                                    max_total_kv_tokens=int(wl.kv_lens.astype(np.int64).sum()), **kw)
        return self.bsra.Engine(cfg, torch.cuda.current_device())

    def plan(self, eng, stream=None):
        i = self.inp0
        eng.plan(i.qo_indptr, i.kv_page_indptr, i.kv_last_page_len, i.sm_scale, stream=stream)

    def run_layer(self, eng, r, stream=None):
        inp, o, lse = self.layers[r]
        eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse,
                stream=stream)


def time_device_steps(L: Layered, eng, steps, warmup, use_graph=True):
    """K timed steps; each = plan() + all layers (one graph replay). Returns per-step ms list."""
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        L.plan(eng, s)
        for r in range(len(L.layers)):
            L.run_layer(eng, r, s)
    torch.cuda.synchronize()
    graph = None
    if use_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            for r in range(len(L.layers)):
                L.run_layer(eng, r, s)
    launches_per_step = eng.last_launches() * len(L.layers)

    def one_step():
        L.plan(eng, s)
        if graph is not None:
            graph.replay()
        else:
            for r in range(len(L.layers)):
                L.run_layer(eng, r, s)

    with torch.cuda.stream(s):
        for _ in range(warmup):
            one_step()
    torch.cuda.synchronize()
    return s, one_step, launches_per_step


def per_launch_ms(L: Layered, eng, reps=3):
    """CUDA events around each run() on its stream (attention + contraction kernels)."""
    s = torch.cuda.Stream()
    evs = []
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        L.plan(eng, s)
        for r in range(len(L.layers)):  # warm pass: first-launch costs stay out of the average
            L.run_layer(eng, r, s)
        for _ in range(reps):
            for r in range(len(L.layers)):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                L.run_layer(eng, r, s)
                b.record(s)
                evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in evs]))


def e2e_steps(L: Layered, eng, steps, warmup):
    """End to end through the public API with HOST buffers. Per step: plan() on the host (Algorithm
    1 + upload), then, for every layer r, H2D of q[r] from pinned memory, run(r), and D2H of o[r]
    and lse[r] into pinned memory, plus the page table's H2D once per step. The copies run on a
    copy stream and overlap the other layers' kernels (event-ordered per layer); the per-step
    sequence of copies and run() calls is captured once in a CUDA graph (the same public calls,
    replayed). KV pools are the resident cache (model state), not per-step input."""
    s = torch.cuda.Stream()
    cp_in, cp_out = torch.cuda.Stream(), torch.cuda.Stream()
    host_q = [inp.q.cpu().pin_memory() for inp, _, _ in L.layers]
    host_idx = L.inp0.kv_page_indices.cpu().pin_memory()
    host_o = [o.cpu().pin_memory() for _, o, _ in L.layers]
    host_l = [l.cpu().pin_memory() for _, _, l in L.layers]
    h2d = sum(q.numel() * q.element_size() for q in host_q) + host_idx.numel() * 4
    d2h = sum(o.numel() * o.element_size() for o in host_o) + sum(l.numel() * 4 for l in host_l)
    n = len(L.layers)

    def body():
        ev_in = [torch.cuda.Event() for _ in range(n)]
        ev_run = [torch.cuda.Event() for _ in range(n)]
        cp_in.wait_stream(s)
        with torch.cuda.stream(cp_in):
            L.inp0.kv_page_indices.copy_(host_idx, non_blocking=True)
            for r, (inp, _, _) in enumerate(L.layers):
                inp.q.copy_(host_q[r], non_blocking=True)
                ev_in[r].record(cp_in)
        for r in range(n):
            s.wait_event(ev_in[r])
            L.run_layer(eng, r, s)
            ev_run[r].record(s)
        with torch.cuda.stream(cp_out):
            for r, (_, o, lse) in enumerate(L.layers):
                cp_out.wait_event(ev_run[r])
                host_o[r].copy_(o, non_blocking=True)
                host_l[r].copy_(lse, non_blocking=True)
        s.wait_stream(cp_out)
        s.wait_stream(cp_in)

    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        L.plan(eng, s)
        body()  # eager warm pass
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        body()

    def step():
        with torch.cuda.stream(s):
            L.plan(eng, s)
            graph.replay()

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(steps):
        step()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps, h2d, d2h


def oracle_cpu_baseline(wl, inp_host, budget_s=12.0):
    """The float64 C oracle, as it stands, on this host's cores: whole configs[1] layers
    repeated until ~budget_s of CPU work. Returns (TB/s of KV, threads, sample text, the first
    run's (o, lse) for the §8(d.6) parity fields)."""
    import oracle
    threads = len(os.sched_getaffinity(0))
    by = decode_bytes(wl)["total"]
    t0 = time.perf_counter()
    n = 0
    first = None
    while True:
        r = oracle.paged_attention(**inp_host, num_threads=threads)
        if first is None:
            first = r
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s or n >= 200:
            break
    return (by * n / el / 1e12, threads, f"{n} full configs[1] layer(s) (batch 128, one layer each) in {el:.1f} s",
            first)


def host_inputs(inp):
    from synth import raw_bits
    wl = inp.wl
    return dict(qo_indptr=inp.qo_indptr, kv_page_indptr=inp.kv_page_indptr, kv_last_page_len=inp.kv_last_page_len,
                kv_page_indices=inp.kv_page_indices.cpu().numpy(), q=raw_bits(inp.q), k_pool=raw_bits(inp.k_pool),
                v_pool=raw_bits(inp.v_pool), k_strides=inp.k_strides, v_strides=inp.v_strides, H_qo=wl.H_qo,
                H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype, mask=wl.mask,
                sm_scale=inp.sm_scale)


def time_graph(fn, s, reps, warmup=3):
    """Capture fn() (a sequence of C-ABI launches on stream s) once; time `reps` replays."""
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    with torch.cuda.stream(s):
        for _ in range(warmup):
            g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def bench_contiguous(dev, pk, reps=9):
    """the page table's cost. The same keys / values as a paged pool
    (permuted 16-token pages, the workload) and as contiguous ragged tensors (BSRA_FLAG_RAGGED_KV),
    per-launch CUDA events (median), configs[1] decode and configs[2] prefill."""
    def timed(fn):
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

    import paper_2501_01005_b200 as bsra
    out = {"unit": "us per launch", "paper": "App. B (P:443-447): <= 1 % decode, ~10 % prefill on H100/FA3"}
    for key, wl, tq in (("decode_c2", synth.c2_decode_llama8b(), 16), ("prefill_c3", synth.c3_prefill_llama70b(), 0)):
        inp = synth.make_inputs(wl, device=dev)
        nq = int(wl.qo_lens.sum())
        kw = dict(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, dtype=wl.dtype, mask=wl.mask, max_batch=wl.batch,
                  max_total_qo_rows=nq, num_ctas=148, tile_q=tq)
        o = torch.empty((nq, wl.H_qo, wl.D), device=dev, dtype=torch.bfloat16)
        lse = torch.empty((nq, wl.H_qo), device=dev)
        pe = bsra.Engine(bsra.make_config(page_size=wl.page_size, **kw), torch.cuda.current_device())
        pe.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
        paged = timed(lambda: pe.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides,
                                     inp.kv_page_indices, o, lse))
        rk = synth.ragged_kv(inp)
        re_ = bsra.Engine(bsra.make_config(page_size=128, ragged_kv=True, **kw), torch.cuda.current_device())
        re_.plan_ragged(inp.qo_indptr, rk.kv_indptr, inp.sm_scale)
        contig = timed(lambda: re_.run_ragged(inp.q, rk.k, rk.v, rk.k_strides, rk.v_strides, o, lse))
        out[key] = {"paged_us": paged, "contiguous_us": contig,
                    "page_table_overhead_pct": 100.0 * (paged / contig - 1.0)}
        if tq == 16:  # decode: the cp.async row gather at B_c = 16 and at B_c = 1 (P:436's setting)
            ce = bsra.Engine(bsra.make_config(page_size=wl.page_size, cp_gather=True, **kw), torch.cuda.current_device())
            ce.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
            out[key]["paged_row_gather4_us"] = timed(lambda: ce.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides,
                                                                    inp.v_strides, inp.kv_page_indices, o, lse))
            ca = bsra.Engine(bsra.make_config(page_size=wl.page_size, cp_gather=True, cp_async=True, **kw),
                             torch.cuda.current_device())
            ca.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
            out[key]["paged_row_cp_async_us"] = timed(lambda: ca.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides,
                                                                     inp.v_strides, inp.kv_page_indices, o, lse))
            import dataclasses
            wl1 = dataclasses.replace(wl, page_size=1)
            i1 = synth.make_inputs(wl1, device=dev)
            e1 = bsra.Engine(bsra.make_config(page_size=1, **kw), torch.cuda.current_device())
            e1.plan(i1.qo_indptr, i1.kv_page_indptr, i1.kv_last_page_len, i1.sm_scale)
            out[key]["paged_page_size_1_us"] = timed(lambda: e1.run(i1.q, i1.k_pool, i1.v_pool, i1.k_strides,
                                                                    i1.v_strides, i1.kv_page_indices, o, lse))
            out[key]["page_size_1_overhead_pct"] = 100.0 * (out[key]["paged_page_size_1_us"] / contig - 1.0)
            out[key]["page_size_1_kernel"] = e1.selected_kernel()
            del ce, ca, i1, e1
        del inp, rk, pe, re_, o, lse
        torch.cuda.empty_cache()
    return out


def bench_fp8_decode(dev, pk, args, world, rank, bf16_ms):
    """the configs[1] decode step with an E4M3 KV cache: same
    lengths, layers, graph and timing as the headline line; bytes counted at one byte per KV
    element. `speedup` = bf16 step time / fp8 step time (same tokens)."""
    import dataclasses
    wl = dataclasses.replace(synth.c2_decode_llama8b(), kv_dtype="e4m3")
    L = Layered(wl, args.layers, dev, seed_base=1000 * rank)
    eng = L.engine(num_ctas=args.num_ctas, tile_q=16, kernel=args.kernel, pdl=not args.no_pdl, max_qo_len=1)
    s, one_step, _ = time_device_steps(L, eng, args.steps, args.warmup, not args.no_graph)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(args.steps):
            one_step()
        b.record(s)
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b) / args.steps, world)
    by = decode_bytes(wl)
    launch_ms = per_launch_ms(L, eng)
    tokens = int(wl.kv_lens.sum()) * args.layers * world
    return {"workload": "c2_decode_llama8b (configs[1]) with an E4M3 KV cache, bf16 q/o", "unit": "TB/s",
            "value": world * by["total"] * args.layers / (ms * 1e-3) / 1e12, "ms_per_step": ms,
            "kv_tokens_per_s": tokens / (ms * 1e-3), "speedup_vs_bf16_kv": bf16_ms / ms,
            "launch_ms": launch_ms, "frac": by["total"] / (launch_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
            "kernel": eng.selected_kernel(), "algorithmic_bytes_per_launch": by["total"]}


def bench_rope_decode(dev, pk, args, world, rank, plain_ms):
    """SURVEY §8(f) NEXT-3 fused RoPE (R31): the configs[1] decode step with q and
    k rotated inside the decode kernel (Llama-3 theta 500000; the cache holds un-rotated keys, as
    StreamingLLM needs). Same layers / graph / timing as the headline; `overhead` = the step time
    relative to the plain step (same bytes)."""
    import dataclasses
    wl = dataclasses.replace(synth.c2_decode_llama8b(), rope_theta=500000.0)
    L = Layered(wl, args.layers, dev, seed_base=1000 * rank)
    eng = L.engine(num_ctas=args.num_ctas, tile_q=16, kernel=args.kernel, pdl=not args.no_pdl, max_qo_len=1)
    s, one_step, _ = time_device_steps(L, eng, args.steps, args.warmup, not args.no_graph)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(args.steps):
            one_step()
        b.record(s)
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(b) / args.steps, world)
    by = decode_bytes(wl)
    launch_ms = per_launch_ms(L, eng)
    return {"workload": "c2_decode_llama8b (configs[1]) with fused RoPE (theta 500000)", "unit": "TB/s",
            "value": world * by["total"] * args.layers / (ms * 1e-3) / 1e12, "ms_per_step": ms,
            "step_time_vs_plain": ms / plain_ms, "launch_ms": launch_ms,
            "frac": by["total"] / (launch_ms * 1e-3) / 1e9 / pk["hbm_gbs"], "kernel": eng.selected_kernel()}


def bench_composable(dev, pk, world=1, rank=0, layers=16, reps=20):
    """configs[3]: 8K shared prefix + 64 branches x 256-token suffixes, one decode step per layer
    through ComposableDecode (prefix engine on tensor-core tiles + suffix engine + ⊕), every layer
    its own pool (16 x 101.7 MB >> L2). Also the single-format baseline the paper compares with
    (64 requests x 528 pages through the decode kernel)."""
    import paper_2501_01005_b200 as bsra
    h0, h1 = local_heads(8, world, rank)  # N > 1: the ranks split the 8 kv heads (no collective)
    cis = [synth.c4_composable(device=dev, seed_base=100 * r + 1000 * rank, H_qo=4 * (h1 - h0), H_kv=h1 - h0)
           for r in range(layers)]
    c0 = cis[0]
    n = c0.q.shape[0]
    # prefix (paired 256-row tiles, tensor-bound) and suffix (HBM-bound) grids run concurrently on
    # 64 + 84 SMs (scripts/composable_perf.py split sweep; PDL measured slower in this mode)
    comp = bsra.ComposableDecode(H_qo=c0.H_qo, H_kv=c0.H_kv, D=c0.D, page_size=c0.page_size, n_branch=n,
                                 prefix_ctas=64, suffix_ctas=84, concurrent=True)
    comp.plan(c0.prefix, c0.suffix, c0.sm_scale)
    pi = torch.from_numpy(c0.prefix["kv_page_indices"]).to(dev)
    si = torch.from_numpy(c0.suffix["kv_page_indices"]).to(dev)
    outs = [(torch.empty((n, c0.H_qo, c0.D), device=dev, dtype=c0.q.dtype), torch.empty((n, c0.H_qo), device=dev))
            for _ in cis]
    s = torch.cuda.Stream()

    def step():
        for ci, (o, l) in zip(cis, outs):
            comp.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, pi, si, o, l, stream=s)

    barrier(world)
    ms = max_over_ranks(time_graph(step, s, reps) / layers, world)
    es = 2
    unique = (8192 + n * 256) * 8 * c0.D * 2 * es + n * 32 * c0.D * es * 2 + n * 32 * 4  # all 8 / 32 heads
    # single format: 64 requests over prefix + own suffix pages (re-reads the prefix per branch)
    cfg = bsra.make_config(H_qo=c0.H_qo, H_kv=c0.H_kv, D=c0.D, page_size=c0.page_size, dtype="bf16", max_batch=n,
                           max_total_qo_rows=n, num_ctas=148, tile_q=16)
    eng = bsra.Engine(cfg, torch.cuda.current_device())
    sg = c0.single
    eng.plan(sg["qo_indptr"], sg["kv_page_indptr"], sg["kv_last_page_len"], c0.sm_scale)
    sgi = torch.from_numpy(sg["kv_page_indices"]).to(dev)

    def step_single():
        for ci, (o, l) in zip(cis, outs):
            eng.run(ci.q, ci.k_pool, ci.v_pool, ci.strides, ci.strides, sgi, o, l, stream=s)

    ms_single = max_over_ranks(time_graph(step_single, s, max(3, reps // 4)) / layers, world)
    tbs = unique / (ms * 1e-3) / 1e12
    return {"workload": "c4_composable (BASELINE configs[3]): 8K prefix + 64 x 256 suffix, 32/8 heads",
            "us_per_layer": ms * 1e3, "unique_bytes_per_layer": unique, "value": tbs, "unit": "TB/s (unique bytes)",
            "frac": tbs * 1e3 / world / pk["hbm_gbs"], "single_format_us_per_layer": ms_single * 1e3,
            "n_gpus": world, "scaling": "strong (kv heads split)" if world > 1 else None,
            "speedup_vs_single_format": ms_single / ms, "launches_per_layer": comp.launches(),
            "kernels": [comp.prefix.selected_kernel(), comp.suffix.selected_kernel(), "merge_states"]}


def bench_long_context(dev, pk, world, rank, local, layers=2, reps=10):
    """configs[4]: 4 requests x 512K tokens, Llama-3-8B heads. The sequence is split across the
    `world` GPUs (rank r owns a contiguous 1/P of every request's pages); each rank runs the
    paged attention of its shard (fp32 state) and the states are combined by the library's NCCL
    all-gather + ⊕ (bsra_dist). Total work fixed -> strong scaling of one long-context step."""
    import paper_2501_01005_b200 as bsra
    full = synth.c5_long_decode()
    # this rank's share of every request (bsra_dist_shard_bsr over the full page table): its
    # lengths decide the shard workload; the shard's own pool holds exactly those pages
    ps = full.page_size
    n_pages = full.num_pages()
    kp = np.concatenate([[0], np.cumsum(n_pages)]).astype(np.int32)
    last = (full.kv_lens - (n_pages - 1) * ps).astype(np.int32)
    ki, _, kl = bsra.sequence_shard(kp, np.arange(int(kp[-1]), dtype=np.int32), last, ps, world, rank)
    nr = ki[1:] - ki[:-1]
    shard_lens = np.where(nr > 0, (nr - 1) * ps + kl, 0).astype(np.int32)
    wl = synth.Workload("c5_shard", full.H_qo, full.H_kv, full.D, full.page_size, full.dtype, "none",
                        full.qo_lens.copy(), shard_lens)
    Ls = [synth.make_inputs(wl, device=dev, seed_base=1000 * rank + 100 * r) for r in range(layers)]
    nq = wl.batch
    # few long rows: plan with the queue count of smallest Algorithm-1 makespan (148 CTAs would cut
    # each 512K row into 4.6 chunks; scripts/long_ctx_ctas.py)
    cfg = bsra.make_config(H_qo=wl.H_qo, H_kv=wl.H_kv, D=wl.D, page_size=wl.page_size, dtype=wl.dtype,
                           o_dtype="f32", max_batch=wl.batch, max_total_qo_rows=nq, num_ctas=148, tile_q=16,
                           balance_ctas=True)
    eng = bsra.Engine(cfg, local)
    i0 = Ls[0]
    eng.plan(i0.qo_indptr, i0.kv_page_indptr, i0.kv_last_page_len, i0.sm_scale)
    if world > 1:
        import torch.distributed as tdist
        obj = [bsra.Dist.unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    else:
        uid = bsra.Dist.unique_id()
    d = bsra.Dist(world, rank, uid, local)
    scratch = d.scratch(nq, wl.H_qo, wl.D, dev)
    o_loc = torch.empty((nq, wl.H_qo, wl.D), device=dev)
    l_loc = torch.empty((nq, wl.H_qo), device=dev)
    o = torch.empty((nq, wl.H_qo, wl.D), device=dev, dtype=torch.bfloat16)
    l = torch.empty((nq, wl.H_qo), device=dev)
    s = torch.cuda.Stream()

    def step():
        for inp in Ls:
            eng.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, i0.kv_page_indices, o_loc, l_loc,
                    stream=s)
            d.allgather_merge(o_loc, l_loc, scratch, o, l, stream=s)

    barrier(world)
    ms = max_over_ranks(time_graph(step, s, reps) / layers, world)
    kv_total = int(full.kv_lens.astype(np.int64).sum()) * full.H_kv * full.D * 2 * 2
    d.close()
    tbs = kv_total / (ms * 1e-3) / 1e12
    return {"workload": f"c5_long_decode (BASELINE configs[4]): 4 x 512K tokens, sequence split over {world} GPU(s)",
            "us_per_layer": ms * 1e3, "kv_bytes_per_layer": kv_total, "value": tbs, "unit": "TB/s (aggregate)",
            "frac_per_gpu": tbs * 1e3 / world / pk["hbm_gbs"], "scaling": "strong", "n_gpus": world,
            "gather_bytes_per_rank": nq * wl.H_qo * (wl.D + 1) * 4, "kernel": eng.selected_kernel()}


# ------------------------------------------------------- sharded secondaries ---
def local_heads(H_kv, world, rank):
    import paper_2501_01005_b200 as bsra
    return bsra.head_shard(H_kv, world, rank)


def head_sharded_wl(wl, world, rank):
    """The workload one rank of a P-way KV-head split holds: kv heads [h0, h1) and their qo heads
    (bsra_dist_head_shard), same lengths. Bytes and flops are linear in heads, so the aggregate
    over ranks is the whole workload's."""
    import dataclasses
    h0, h1 = local_heads(wl.H_kv, world, rank)
    return dataclasses.replace(wl, H_qo=(h1 - h0) * wl.g, H_kv=h1 - h0), (h0, h1)


def bench_decode_head_sharded(dev, pk, args, world, rank):
    """configs[1] with the FIXED batch of 128 split by KV head over the ranks (strong scaling, no
    collective: the output stays head-sharded, as in tensor-parallel attention). Same graph,
    layers and timing as the headline; aggregate TB/s = whole-step bytes / max-over-ranks time."""
    full = synth.c2_decode_llama8b()
    wl, (h0, h1) = head_sharded_wl(full, world, rank)
    L = Layered(wl, args.layers, dev, seed_base=1000 * rank)
    eng = L.engine(num_ctas=args.num_ctas, tile_q=16, kernel=args.kernel, pdl=not args.no_pdl, max_qo_len=1)
    s, one_step, _ = time_device_steps(L, eng, args.steps, args.warmup, not args.no_graph)
    barrier(world)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(args.steps):
            one_step()
        b.record(s)
    torch.cuda.synchronize()
    mine = a.elapsed_time(b) / args.steps
    per_rank = gather_over_ranks(mine, world)
    ms = max(per_rank)
    step_bytes = decode_bytes(full)["total"] * args.layers
    return {"workload": "c2_decode_llama8b (configs[1]), batch 128 fixed, KV heads split over ranks",
            "scaling": "strong", "n_gpus": world, "kv_heads_rank0": [0, local_heads(full.H_kv, world, 0)[1]],
            "value": step_bytes / (ms * 1e-3) / 1e12, "unit": "TB/s (aggregate)", "ms_per_step": ms,
            "per_rank_ms": per_rank, "frac_per_gpu": step_bytes / (ms * 1e-3) / 1e9 / world / pk["hbm_gbs"]}


def bench_prefill(dev, pk, args, world, rank):
    """configs[2] ragged causal prefill, TFLOP/s over visible pairs. N > 1: KV heads split over the
    ranks (8 kv heads; strong scaling), aggregate = whole-layer flops / max-over-ranks time."""
    full = synth.c3_prefill_llama70b()
    wl, _ = head_sharded_wl(full, world, rank) if world > 1 else (full, (0, full.H_kv))
    L3 = Layered(wl, 2, dev, seed_base=1000 * rank)
    e3 = L3.engine(num_ctas=args.num_ctas, kernel=args.kernel, tile_q=args.prefill_tile, pdl=True)
    iso_ms = max(gather_over_ranks(per_launch_ms(L3, e3, reps=3), world))
    # as the decode headline: layers back to back in a CUDA graph with PDL (a layer's prologue and
    # K/V streaming overlap the previous layer's tail); 4 runs (2 layers x 2) per replay
    s = torch.cuda.Stream()

    def four():
        for r in (0, 1, 0, 1):
            L3.run_layer(e3, r, s)
    mine = time_graph(four, s, 5) / 4
    per_rank = gather_over_ranks(mine, world)
    p_ms = max(per_rank)
    fl = causal_flops(full)
    tf = fl / (p_ms * 1e-3) / 1e12
    out = {"value": tf, "unit": "TFLOP/s", "workload": "c3_prefill_llama70b (configs[2])", "n_gpus": world,
           "scaling": "strong" if world > 1 else None, "ms_per_layer": p_ms, "per_rank_ms": per_rank,
           "how": "ms per layer in a CUDA graph of 4 PDL runs over 2 layers (attention + contraction launches)",
           "ms_per_layer_isolated": iso_ms, "value_isolated": fl / (iso_ms * 1e-3) / 1e12,
           "frac": tf / world / pk["bf16_tflops"], "peak": pk["bf16_tflops"], "peak_kind": "burst (measured)",
           "frac_of_sustained": tf / world / pk.get("bf16_tflops_sustained", pk["bf16_tflops"]),
           "kernel": e3.selected_kernel(), "tile_q": int(e3.export_plan()[3]), "flops_per_layer": fl}
    del L3, e3
    torch.cuda.empty_cache()
    if not args.no_fp8:  # the same prefill with an E4M3 KV cache (NEXT-2): gather pass + tcgen05 prefill
        import dataclasses
        L3f = Layered(dataclasses.replace(wl, kv_dtype="e4m3"), 2, dev, seed_base=1000 * rank)
        e3f = L3f.engine(num_ctas=args.num_ctas, kernel=args.kernel, tile_q=args.prefill_tile)
        pf_ms = max(gather_over_ranks(per_launch_ms(L3f, e3f, reps=3), world))
        out["fp8_kv"] = {"ms_per_layer": pf_ms, "value": fl / (pf_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                         "kernel": e3f.selected_kernel(), "launches_per_run": e3f.last_launches(),
                         "vs_bf16_kv": p_ms / pf_ms}
        del L3f, e3f
        torch.cuda.empty_cache()
    return out


def bench_scheduler(dev, pk, args):
    """§8(d.6) scheduler fields on configs[1] (one layer): bsra_plan host time (median of 100 calls)
    and plan + upload (plan, then a stream sync), the Algorithm-1 cost-model efficiency
    (mean / makespan of per-CTA cost), and the balance ablation — the kernel-level analogue of the
    paper's load-balancing study: Algorithm 1 (split KV, 148 persistent CTAs) vs the
    same kernel without KV splitting (LPT over 148 CTAs) vs one (request, kv head) row per CTA
    (non-persistent grid, the FA2-style baseline). Also for a configs[4] shard (4 x 64K tokens),
    where splitting decides whether more than 32 CTAs have work."""
    import dataclasses
    out = {}
    for key, wl in (("c2", synth.c2_decode_llama8b()),
                    ("c5_shard_64k", dataclasses.replace(synth.c5_long_decode(kv_len=65536), name="c5_shard"))):
        L = Layered(wl, 1, dev)
        by = decode_bytes(wl)["total"]
        rows = wl.batch * wl.H_kv
        res = {}
        for name, kw in (("algorithm1", dict(num_ctas=args.num_ctas)),
                         ("algorithm1_queue_balanced", dict(num_ctas=args.num_ctas, balance_ctas=True)),
                         ("no_split_lpt", dict(num_ctas=args.num_ctas, kv_chunk_min=1 << 30)),
                         ("row_per_cta", dict(num_ctas=rows, kv_chunk_min=1 << 30))):
            eng = L.engine(tile_q=16, kernel=args.kernel, **kw)
            ms = per_launch_ms(L, eng, reps=5)
            costs, mk = eng.plan_stats()
            res[name] = {"us_per_launch": ms * 1e3, "TB/s": by / (ms * 1e-3) / 1e12,
                         "frac": by / (ms * 1e-3) / 1e9 / pk["hbm_gbs"], "num_ctas": int(costs.size),
                         "cost_model_efficiency": float(costs.mean() / mk) if mk else None}
            if name == "algorithm1":
                i = L.inp0
                ts = []
                for _ in range(100):
                    t0 = time.perf_counter()
                    eng.plan(i.qo_indptr, i.kv_page_indptr, i.kv_last_page_len, i.sm_scale)
                    ts.append(time.perf_counter() - t0)
                tu = []
                st = torch.cuda.current_stream()
                for _ in range(20):
                    t0 = time.perf_counter()
                    eng.plan(i.qo_indptr, i.kv_page_indptr, i.kv_last_page_len, i.sm_scale)
                    st.synchronize()
                    tu.append(time.perf_counter() - t0)
                res[name]["plan_host_us_median"] = float(np.median(ts)) * 1e6
                res[name]["plan_plus_upload_us_median"] = float(np.median(tu)) * 1e6
                res[name]["plan_words"] = int(eng.export_plan().size)
            del eng
        res["speedup_vs_no_split"] = res["no_split_lpt"]["us_per_launch"] / res["algorithm1"]["us_per_launch"]
        res["speedup_vs_row_per_cta"] = res["row_per_cta"]["us_per_launch"] / res["algorithm1"]["us_per_launch"]
        out[key] = res
        del L
        torch.cuda.empty_cache()
    return out


def bench_quest(dev, pk):
    """SURVEY §8(f) NEXT-4 Quest workload: fine-grained block-sparse decode,
    block 16, 32/32 heads, d 128, batch 1; each head keeps `page_budget` pages of its seq_len/16
    (synth.quest_decode). Per-launch latency (median of 9, CUDA events) through the decode
    kernel; the paper's H100 latencies quoted as context, not as a target. Timed as a CUDA graph of
    20 back-to-back launches (PDL) ÷ 20, so host enqueue cost is out of the figure; `us_serialised`
    is the same without PDL (no overlap between consecutive launches)."""
    paper_h100_us = {(4096, 64): 20.299, (4096, 256): 44.383, (32768, 64): 22.371, (32768, 512): 68.478}
    out = {"unit": "us per launch", "paper": "FlashInfer on H100 SXM5, Table eval-sparsity-flashinfer"}
    for (S, P), ref in paper_h100_us.items():
        wl, extra = synth.quest_decode(S, P)
        inp = synth.make_inputs(wl, device=dev, extra_pages=extra)
        import paper_2501_01005_b200 as bsra
        cfg = bsra.make_config(H_qo=1, H_kv=1, D=128, page_size=16, dtype="bf16", max_batch=wl.batch,
                               max_total_qo_rows=wl.batch, num_ctas=148, tile_q=16, max_qo_len=1, pdl=True)
        e = bsra.Engine(cfg, torch.cuda.current_device())
        o = torch.empty((wl.batch, 1, 128), device=dev, dtype=torch.bfloat16)
        lse = torch.empty((wl.batch, 1), device=dev)
        e.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)
        s = torch.cuda.Stream()

        def twenty():
            for _ in range(20):
                e.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse,
                      stream=s)
        us = time_graph(twenty, s, 10) / 20 * 1e3
        # the same 20 launches without PDL: fully serialised, so no overlap of one launch's
        # prologue / loads with the previous one's tail (the per-kernel latency the paper quotes)
        cfg.flags &= ~bsra.FLAG_PDL
        e2 = bsra.Engine(cfg, torch.cuda.current_device())
        e2.plan(inp.qo_indptr, inp.kv_page_indptr, inp.kv_last_page_len, inp.sm_scale)

        def twenty_serial():
            for _ in range(20):
                e2.run(inp.q, inp.k_pool, inp.v_pool, inp.k_strides, inp.v_strides, inp.kv_page_indices, o, lse,
                       stream=s)
        us_serial = time_graph(twenty_serial, s, 10) / 20 * 1e3
        by = decode_bytes(wl)["total"]
        out[f"seq{S}_budget{P}"] = {"us": us, "TB/s": by / (us * 1e-6) / 1e12, "us_serialised": us_serial,
                                    "bytes": by, "paper_h100_us": ref, "kernel": e.selected_kernel()}
        del inp, e, e2
        torch.cuda.empty_cache()
    return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_single_thread():
    """§8(d.5): the oracle on ONE host thread for configs[0] (best of 3) and one full configs[1]
    layer (one run)."""
    import oracle
    out = {}
    c1 = synth.make_inputs(synth.c1_tiny_decode(), device="cpu")
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        oracle.paged_attention(**host_inputs(c1), num_threads=1)
        ts.append(time.perf_counter() - t0)
    out["c1_us"] = min(ts) * 1e6
    c2 = synth.make_inputs(synth.c2_decode_llama8b(), device="cpu")
    t0 = time.perf_counter()
    oracle.paged_attention(**host_inputs(c2), num_threads=1)
    el = time.perf_counter() - t0
    out["c2_layer_s"] = el
    out["c2_TB/s"] = decode_bytes(c2.wl)["total"] / el / 1e12
    return out


# -------------------------------------------------------------------- main ---
def free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def maybe_relaunch(args):
    """`bench.py --gpus N` without torchrun: re-launch this script under torchrun with N ranks
    (one per GPU) and pass rank 0's JSON line through. Fails loudly if fewer GPUs are visible."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    if args.impl != "reference" and os.environ.get("BSRA_BENCH_ONE_GPU") != "1":
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
            sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    r = subprocess.run(cmd, stdout=subprocess.PIPE)
    _JSON_OUT.write(r.stdout.decode())
    _JSON_OUT.flush()
    sys.exit(r.returncode)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # BSRA_BENCH_ONE_GPU=1 (tests only): every rank on cuda:0 with a gloo group, to exercise the
        # multi-rank code paths on a one-GPU box (the NCCL-based long-context line needs --no-long)
        one_gpu = os.environ.get("BSRA_BENCH_ONE_GPU") == "1"
        backend = "gloo" if args.impl == "reference" or one_gpu else "nccl"
        if torch.cuda.is_available() and args.impl != "reference":
            torch.cuda.set_device(0 if one_gpu else local)
            local = 0 if one_gpu else local
        dist.init_process_group(backend=backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def gather_over_ranks(x: float, world: int) -> list:
    """Every rank's value (device-timed ms), rank order."""
    if world == 1:
        return [x]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, float(x))
    return out


def max_over_ranks(x: float, world: int) -> float:
    return max(gather_over_ranks(x, world))


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def headline_config(world, layers, num_ctas, graph):
    return {"workload": "c2_decode_llama8b (BASELINE configs[1])", "model": "Llama-3-8B attention shape (32/8 heads, d 128)",
            "global_batch": 128 * world, "seq_len": "kv 128-4096 ShareGPT-like (sum 151,721 per 128 requests), l_qo 1",
            "page_size": 16, "layers_per_step": layers, "num_ctas": num_ctas,
            "parallelism": f"requests sharded x{world} (data parallel, no collective)",
            "l2": "inputs larger than L2 (621 MB KV per layer > 126 MB L2); no flush", "graph": graph}


def run_reference(args, world, rank):
    """--impl reference: the oracle (the CPU baseline program) on this host, same metric/config."""
    if rank != 0:
        return
    wl = synth.c2_decode_llama8b()
    inp = synth.make_inputs(wl, device="cpu")
    hin = host_inputs(inp)
    import oracle
    threads = len(os.sched_getaffinity(0))
    # each step = a bounded sample of the workload: 32 of the 128 requests, one layer
    reqs = list(range(0, wl.batch, 4))
    sub = synth.Workload(wl.name, wl.H_qo, wl.H_kv, wl.D, wl.page_size, wl.dtype, wl.mask, wl.qo_lens[reqs],
                         wl.kv_lens[reqs])
    by = decode_bytes(sub)["total"]
    for _ in range(args.warmup):
        oracle.paged_attention(**hin, req_list=reqs, num_threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.paged_attention(**hin, req_list=reqs, num_threads=threads)
    el = (time.perf_counter() - t0) / args.steps
    val = by / el / 1e12
    sample = "requests 0,4,...,124 (32 of 128) of configs[1], one layer per step"
    emit({
        "impl": "reference", "metric": METRIC,
        "value": val, "unit": "TB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": headline_config(world, 1, 0, False),
        "cpu_baseline": {"value": val, "unit": "TB/s", "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": val, "unit": "TB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="bsra", choices=["bsra", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--num-ctas", type=int, default=148)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true")
    ap.add_argument("--prefill-tile", type=int, default=0, help="force T_q for the prefill line (0 = heuristic)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-composable", action="store_true")
    ap.add_argument("--no-contiguous", action="store_true", help="skip the paged-vs-contiguous KV line")
    ap.add_argument("--no-long", action="store_true")
    ap.add_argument("--no-fp8", action="store_true", help="skip the fp8 (E4M3) KV-cache decode line")
    ap.add_argument("--no-sched", action="store_true", help="skip the scheduler / balance-ablation fields")
    ap.add_argument("--no-pdl", action="store_true")
    ap.add_argument("--no-quest", action="store_true", help="skip the Quest block-sparse decode line")
    ap.add_argument("--no-rope", action="store_true", help="skip the fused-RoPE decode line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    maybe_relaunch(args)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    import paper_2501_01005_b200 as bsra
    bsra.lib()  # fail loudly if the extension is missing
    dev = torch.device(f"cuda:{torch.cuda.current_device()}")
    pk, pk_kind = peaks()

    # ---- configs[1]: batched paged decode, Llama-3-8B heads, batch 128 per rank
    wl = synth.c2_decode_llama8b()
    L = Layered(wl, args.layers, dev, seed_base=1000 * rank)
    # consecutive layers are independent -> programmatic dependent launch between them
    eng = L.engine(num_ctas=args.num_ctas, tile_q=16, kernel=args.kernel, pdl=not args.no_pdl, max_qo_len=1)
    by = decode_bytes(wl)
    s, one_step, launches_per_step = time_device_steps(L, eng, args.steps, args.warmup, not args.no_graph)
    clk = ClockSampler(local)
    clk.start()
    barrier(world)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(args.steps):
            one_step()
        b.record(s)
    torch.cuda.synchronize()
    barrier(world)
    clocks = clk.stop()
    per_rank = gather_over_ranks(a.elapsed_time(b) / args.steps, world)
    ms = max(per_rank)
    step_bytes = by["total"] * args.layers
    value = world * step_bytes / (ms * 1e-3) / 1e12

    # ---- roofline of the dominant (and only) kernel: one run() = one persistent tc_decode launch
    # (the contraction is fused in-kernel for decode engines). Its average launch duration over the
    # timed region = the region's CUDA-event time / the launches in it (PDL lets consecutive layers
    # overlap their prologue / tail, so this is what a launch costs inside the step); the isolated
    # figure (events around each run(), launches serialised) is reported beside it.
    region_launch_ms = ms / args.layers
    launch_ms = per_launch_ms(L, eng)
    achieved = by["total"] / (region_launch_ms * 1e-3) / 1e9
    traffic = None
    traffic_src = None
    for fn, key in (("r02d_ncu_traffic.json", "tc_decode"), ("r02c_ncu_traffic.json", "tc_decode")):
        try:  # DRAM read+write per launch from the committed ncu --set full capture of this kernel
            with open(os.path.join(ROOT, "profiles", fn)) as f:
                traffic = json.load(f)[key]["traffic_bytes"]
            traffic_src = f"profiles/{fn} (ncu --set full, one launch)"
            break
        except Exception:
            pass
    roof = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / pk["hbm_gbs"], "traffic": traffic, "peak_kind": pk_kind,
            "kernel": f"bsra {eng.selected_kernel()} (one launch per run(), contraction fused)",
            "algorithmic_bytes_per_launch": by["total"], "launch_ms": region_launch_ms,
            "launch_ms_how": "timed region / launches in it (32 per step, PDL graph; includes the plan upload)",
            "launch_ms_isolated": launch_ms, "frac_isolated": by["total"] / (launch_ms * 1e-3) / 1e9 / pk["hbm_gbs"],
            "traffic_source": traffic_src}

    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e_ms, h2d, d2h = e2e_steps(L, eng, max(3, args.steps // 4), 2)
        e2e_ms = max_over_ranks(e2e_ms, world)
        e2e = {"value": world * step_bytes / (e2e_ms * 1e-3) / 1e12, "unit": "TB/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
               "how": "per step: plan() on host, then one graph replay of {H2D q[r] (copy stream) -> run(r) -> "
                      "D2H o[r], lse[r] (copy stream)} for every layer r, copies overlapping other layers' kernels"}
    # determinism and the §8(d.6) parity inputs: layer 0 run twice (bitwise equal), its output and plan
    inp0, o0, l0 = L.layers[0]
    outs = []
    for _ in range(2):
        o0.fill_(float("nan"))
        L.run_layer(eng, 0)
        torch.cuda.synchronize()
        outs.append((o0.clone(), l0.clone()))
    head_check = {"deterministic": bool(torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])),
                  "o": outs[1][0].float().cpu().numpy(), "lse": outs[1][1].cpu().numpy(), "plan": eng.export_plan()}
    # layer 0's own inputs on the host for the oracle leg (the CPU and CUDA generators differ)
    head_inputs = host_inputs(inp0) if rank == 0 and world == 1 and not args.no_cpu_baseline else None
    del L, eng, outs
    torch.cuda.empty_cache()

    # ---- secondary: configs[1] with the batch fixed and KV heads split over the ranks (N > 1)
    head_sharded = None
    if world > 1:
        head_sharded = bench_decode_head_sharded(dev, pk, args, world, rank)
        torch.cuda.empty_cache()

    # ---- secondary: the same decode step with an fp8 (E4M3) KV cache (NEXT-2)
    fp8 = None
    if not args.no_fp8:
        fp8 = bench_fp8_decode(dev, pk, args, world, rank, ms)
        torch.cuda.empty_cache()

    # ---- secondary: the same decode step with fused RoPE (NEXT-3)
    rope = None
    if not args.no_rope:
        rope = bench_rope_decode(dev, pk, args, world, rank, ms)
        torch.cuda.empty_cache()

    # ---- secondary: configs[2] ragged causal prefill TFLOP/s (one layer, per-launch events)
    prefill = None
    if not args.no_prefill:
        prefill = bench_prefill(dev, pk, args, world, rank)
        torch.cuda.empty_cache()

    composable = None
    if not args.no_composable:
        composable = bench_composable(dev, pk, world, rank)
        torch.cuda.empty_cache()

    contiguous = None
    if not args.no_contiguous and world == 1:
        contiguous = bench_contiguous(dev, pk)
        torch.cuda.empty_cache()

    sched = None
    if not args.no_sched and world == 1:
        sched = bench_scheduler(dev, pk, args)
        torch.cuda.empty_cache()

    quest = None
    if not args.no_quest and world == 1:
        quest = bench_quest(dev, pk)
        torch.cuda.empty_cache()

    long_ctx = None
    if not args.no_long:
        long_ctx = bench_long_context(dev, pk, world, rank, local)
        torch.cuda.empty_cache()

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, th, sample, ref = oracle_cpu_baseline(wl, head_inputs)
        cpu = {"value": v, "unit": "TB/s", "cores": th, "kind": "oracle", "sample": sample, "cpu_model": cpu_model(),
               "single_thread": oracle_single_thread()}
        # §8(d.6) parity fields from the same oracle run: the headline layer 0 (same seeds) vs the
        # float64 oracle on every row, and the headline plan vs the Python Algorithm 1 (bit-exact)
        from oracle import scheduler_ref
        fin = np.isfinite(ref[1])
        ref_plan = scheduler_ref.plan_ref(wl.qo_lens, wl.kv_lens, g=wl.g, H_kv=wl.H_kv, num_ctas=args.num_ctas,
                                          align=wl.page_size, T_q=16, qo_begin=head_inputs["qo_indptr"][:-1],
                                          page_begin=head_inputs["kv_page_indptr"][:-1])
        parity = {"workload": "configs[1] layer 0, all 128 x 32 rows, vs the float64 oracle",
                  "max_abs_do": float(np.max(np.abs(head_check["o"] - ref[0]))),
                  "max_abs_dlse": float(np.max(np.abs(head_check["lse"][fin] - ref[1][fin]))),
                  "tolerance": {"o": 1e-2, "lse": 1e-3},
                  "plan_bit_exact_vs_python_algorithm1": bool(np.array_equal(head_check["plan"], ref_plan.image)),
                  "deterministic_run_to_run": head_check["deterministic"]}

    if rank == 0:
        out = {
            "metric": METRIC,
            "value": value, "unit": "TB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "per_rank_ms": per_rank, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": headline_config(world, args.layers, args.num_ctas, not args.no_graph),
            "frac_of_hbm_peak": value / world * 1e3 / pk["hbm_gbs"],
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "prefill": prefill,
            "decode_head_sharded": head_sharded, "composable": composable, "long_context": long_ctx,
            "contiguous_kv": contiguous, "decode_fp8": fp8, "scheduler": sched, "quest": quest,
            "decode_rope": rope, "parity": parity,
            "gpu_launches": launches_per_step * args.steps, "clocks": clocks,
        }
        emit(out)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
