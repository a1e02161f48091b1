#!/usr/bin/env python3
"""AOR (include/ckpt_aor.h, PAPER.md P.494-505) at the paper's scale, one process per GPU.

  torchrun --nproc-per-node 4 tools/aor_bench.py              # 7B ZeRO-1 over m = 4 GPUs
  python tools/aor_bench.py --params 1000000000                 # m = 1

Per step and member: the complete flat gradient is redrawn on the device (the backward
pass), ckpt_aor_step + ckpt_aor_fence are issued on the training stream, the owner applies
its own Eq 4 update on the device, and the host replica of the next member's shard is
updated by the library's worker.  Reported (max over ranks, median over steps):
  - fence_ms: training stream blocked until the step's gradient slice left the GPU
              (copy engine, D2H GB/s = slice bytes / fence time)
  - replica_ms: ckpt_aor_step call -> replica CLEAN at that step (host wall)
  - host update GB/s: Eq 4 bytes (read g, read w, write w) / worker time in Eq 4
  - host roofline: the same routine (ckpt_aor_apply) on T threads over resident host
    buffers, all ranks at once -- the host-memory bandwidth the update can reach
  - gemm slowdown: bf16 8192^3 GEMMs on the training stream while a step is in flight
and a sampled bit-exact check of every replica against the oracle's Eq 4.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def host_roofline(C, np, n_elems, threads, reps=3):
    """GB/s of the library's Eq 4 routine on `threads` threads over host buffers."""
    w = np.ones(n_elems, np.float32)
    g = np.full(n_elems, 1e-3, np.float32)
    per = -(-n_elems // threads)
    best = 0.0
    for _ in range(reps):
        th = []
        t0 = time.perf_counter()
        for i in range(threads):
            lo, hi = i * per, min(n_elems, (i + 1) * per)
            th.append(threading.Thread(target=C.ckpt_aor_apply, args=(w[lo:hi], g[lo:hi], 1e-3)))
        for t in th:
            t.start()
        for t in th:
            t.join()
        dt = time.perf_counter() - t0
        best = max(best, 12.0 * n_elems / dt / 1e9)
    return best


def run_config(a, C, np, torch, oracle, bar, amax, amin, key, chunk_mib, threads, roof, default_threads,
               m, me, P, bounds, owner, n_rep, esz, gen, master, grad, local, dev, s0, gemms, rank):
    opt = C.ckpt_aor_options_default(key=key, chunk_bytes=chunk_mib << 20, n_slots=a.n_slots, threads=threads,
                                     grad_dtype=C.CKPT_DTYPE_BF16 if a.bf16 else C.CKPT_DTYPE_FP32)
    t0 = time.perf_counter()
    ctx = C.ckpt_aor_create(local, opt, master, grad, bounds, me)
    create_s = time.perf_counter() - t0
    bar()
    C.ckpt_aor_seed(ctx, 0)
    bar()
    # sampled oracle replica of the held shard: the replica at the sampled indices after the seed
    rng = np.random.default_rng(7 + me)
    idx = np.sort(rng.choice(n_rep, size=min(a.samples, n_rep), replace=False)) if n_rep else np.zeros(0, np.int64)
    rep_s, _, _ = C.ckpt_aor_view(ctx, copy=False)
    want = rep_s[idx].copy()
    idx_t = torch.from_numpy(idx).to(dev) + bounds[owner]
    rows = []
    for it in range(a.warmup + a.steps):
        eta = 1e-3 * (1 + it)
        grad.normal_(0.0, 1e-3, generator=gen)          # backward: the complete gradient
        torch.cuda.synchronize()
        bar()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tw0 = time.perf_counter()
        e0.record(s0)
        sid = C.ckpt_aor_step(ctx, eta, s0)
        C.ckpt_aor_fence(ctx, sid, s0)
        e1.record(s0)
        g_s = grad[idx_t]                                # the sampled gradient (after the fence)
        master.sub_(grad[bounds[me]:bounds[me + 1]].float() * eta)   # the owner's own update
        C.ckpt_aor_wait(ctx, sid)
        tw1 = time.perf_counter()
        s0.synchronize()
        gs = g_s.view(torch.int16).cpu().numpy().view(np.uint16) if a.bf16 else g_s.cpu().numpy()
        want = oracle.aor_update(want, gs, eta)
        if it >= a.warmup:
            rows.append({"fence_ms": e0.elapsed_time(e1), "replica_ms": (tw1 - tw0) * 1e3})
    st = C.ckpt_aor_get_stats(ctx)
    got, step, state = C.ckpt_aor_view(ctx, copy=False)
    ok = bool(np.array_equal(got[idx].view(np.uint32), want.view(np.uint32))) and state == C.CKPT_AOR_CLEAN
    okall = amax(0.0 if ok else 1.0) == 0.0

    corun = None
    if not a.no_corun:
        # interleaved A/B x3: GEMMs alone, then GEMMs while one AOR step is in flight (the
        # GEMM window covers the D2H phase and the start of the host phase); medians
        gemms(20)
        torch.cuda.synchronize()
        alone, withs = [], []
        for _ in range(3):
            e = gemms(40)
            torch.cuda.synchronize()
            alone.append(e[0].elapsed_time(e[1]) / 40)
            grad.normal_(0.0, 1e-3, generator=gen)
            torch.cuda.synchronize()
            bar()
            sid = C.ckpt_aor_step(ctx, 1e-4, s0)
            e = gemms(40)
            C.ckpt_aor_fence(ctx, sid, s0)
            torch.cuda.synchronize()
            C.ckpt_aor_wait(ctx, sid)
            withs.append(e[0].elapsed_time(e[1]) / 40)
        ga, gw = statistics.median(alone), statistics.median(withs)
        corun = {"gemm_ms_alone": round(ga, 3), "gemm_ms_during_aor": round(gw, 3),
                 "slowdown_pct_max_over_ranks": round(amax(100.0 * (gw / ga - 1)), 2)}

    fence = amax(statistics.median(r["fence_ms"] for r in rows))
    repl = amax(statistics.median(r["replica_ms"] for r in rows))
    bpe = 10.0 if a.bf16 else 12.0                       # read g + read w + write w
    upd_gbs = amin(bpe * n_rep * st["steps"] / max(st["update_s"], 1e-9) / 1e9)
    rec = {"tool": "aor_bench", "m": m, "params": P, "grad_dtype": "bf16" if a.bf16 else "fp32",
           "shard_elems": n_rep, "grad_slice_bytes": n_rep * esz, "chunk_mib": chunk_mib, "n_slots": a.n_slots,
           "host_threads_per_rank": threads, "steps": a.steps,
           "fence_ms": round(fence, 2), "d2h_gbs_per_gpu": round(n_rep * esz / (fence / 1e3) / 1e9, 2),
           "replica_ms": round(repl, 2),
           "replica_elems_per_s_per_gpu": round(n_rep / (repl / 1e3) / 1e9, 3),
           "host_update_gbs_per_rank": round(upd_gbs, 2),
           "host_roofline_gbs_per_rank": round(amin(roof), 2), "host_roofline_threads": default_threads,
           "host_update_frac": round(upd_gbs / amin(roof), 3) if roof else None,
           # the whole step against host DRAM: D2H write + Eq 4 (esz + bpe bytes per element)
           # at this rank's share of the all-ranks routine bandwidth
           "replica_roofline_ms": round((esz + bpe) * n_rep / (amin(roof) * 1e9) * 1e3, 2) if roof else None,
           "replica_roofline_frac": round((esz + bpe) * n_rep / (amin(roof) * 1e9) * 1e3 / repl, 3) if roof else None,
           "stall_s_rank0": round(st["stall_s"], 3), "create_s_rank0": round(create_s, 2),
           "bit_exact_sampled": okall, "samples_per_rank": int(idx.size), "gemm_corun": corun}
    if rank == 0:
        print(json.dumps(rec), flush=True)
    C.ckpt_aor_destroy(ctx)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--params", type=int, default=6_738_415_616, help="flat parameter count (Llama-2-7B)")
    p.add_argument("--bf16", action="store_true", help="bf16 gradients (fp32 default)")
    p.add_argument("--steps", type=int, default=4)
    p.add_argument("--warmup", type=int, default=1)
    p.add_argument("--chunk-mib", default="16", help="comma list: one configuration each")
    p.add_argument("--n-slots", type=int, default=0)
    p.add_argument("--threads", default="", help="comma list of host threads per rank (default min(8, cores/2m))")
    p.add_argument("--samples", type=int, default=1 << 20)
    p.add_argument("--no-corun", action="store_true")
    a = p.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2310_12670_b200 import ckpt as C

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def bar():
        if world > 1:
            dist.barrier()

    def amax(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def amin(x):
        return -amax(-x)

    m, me = world, rank
    P = a.params
    bounds = [(P * j // m) // 64 * 64 if j < m else P for j in range(m + 1)]
    n_me = bounds[me + 1] - bounds[me]
    owner = (me + 1) % m
    n_rep = bounds[owner + 1] - bounds[owner]
    gdt = torch.bfloat16 if a.bf16 else torch.float32
    esz = 2 if a.bf16 else 4
    gen = torch.Generator(device=dev).manual_seed(1234)   # the same stream on every rank
    master_gen = torch.Generator(device=dev).manual_seed(99 + me)
    master = torch.empty(n_me, device=dev).normal_(generator=master_gen)
    grad = torch.empty(P, device=dev, dtype=gdt)
    default_threads = max(1, min(8, (os.cpu_count() or 8) // (2 * m)))
    bar()
    roof = host_roofline(C, np, 1 << 27, default_threads)  # 512 MiB per rank, all ranks at once
    bar()
    key = C.aor_group_key()
    A = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    B = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
    hp = torch.cuda.Stream(priority=-1)

    def gemms(n):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(hp):
            ev0.record()
            for _ in range(n):
                torch.matmul(A, B)
            ev1.record()
        return ev0, ev1

    s0 = torch.cuda.current_stream()
    for chunk_mib in [int(x) for x in a.chunk_mib.split(",")]:
        for threads in ([int(x) for x in a.threads.split(",")] if a.threads else [default_threads]):
            run_config(a, C, np, torch, oracle, bar, amax, amin, key, chunk_mib, threads, roof, default_threads,
                       m, me, P, bounds, owner, n_rep, esz, gen, master, grad, local, dev, s0, gemms, rank)
            key += 2
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
