#!/usr/bin/env python3
"""HAS placement on B200 (Alg 1 layers, P.419-425), N=1: a training-like loop alternates a
compute-bound phase (bf16 GEMMs) and an HBM-bound phase (an Adam-like streaming update);
a C2 snapshot runs meanwhile (a) ungated or (b) with its D2H confined to the compute
phases by ckpt_window (CKPT_OPT_WINDOWED).  Reports each phase's mean time with no
snapshot, ungated and gated, and the snapshot's duration."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2310_12670_b200 import ckpt as C  # noqa: E402
from synth.gpu import descriptors, make_rank_state  # noqa: E402

dev = torch.device("cuda", 0)
specs, ts = make_rank_state("c2_7b_tp8", 0, dev)
n = 8192
A = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
B = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
P = torch.randn(512 << 20, dtype=torch.float32, device=dev)  # 2 GiB "params"
M = torch.randn_like(P)
V = torch.rand_like(P)
T = torch.cuda.Stream(device=dev, priority=-5)


def iteration(ctx, gated, evs):
    with torch.cuda.stream(T):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        if gated:
            C.ckpt_window(ctx, True, T)
        e0.record(T)
        for _ in range(6):
            torch.matmul(A, B)
        e1.record(T)
        if gated:
            C.ckpt_window(ctx, False, T)
        for _ in range(2):  # HBM-bound: p -= 1e-3 * m / (sqrt(v) + 1e-8)
            P.addcdiv_(M, V.sqrt().add_(1e-8), value=-1e-3)
        e2.record(T)
        evs.append((e0, e1, e2))


def run(mode, iters):
    """Median phase times over `iters` iterations issued right after the snapshot starts
    (sized so the snapshot is in flight for all of them)."""
    ctx = None
    if mode != "none":
        flags = C.CKPT_OPT_TIMING | (C.CKPT_OPT_WINDOWED if mode == "gated" else 0)
        ctx = C.ckpt_create(0, C.ckpt_options_default(n_slots=0, bucket_bytes=256 << 20, flags=flags))
        C.ckpt_register(ctx, descriptors(ts, specs))
        C.ckpt_protect(ctx, 1, 0)
        sid = C.ckpt_snapshot(ctx, 0, T)  # warm-up snapshot (window open)
        C.ckpt_wait(ctx, sid)
    for _ in range(3):
        iteration(ctx, False, [])
    torch.cuda.synchronize()
    evs = []
    t0 = time.perf_counter()
    sid = C.ckpt_snapshot(ctx, 0, T) if ctx else None
    for i in range(iters):
        iteration(ctx, mode == "gated", evs)
    snap_s = None
    if ctx:
        if mode == "gated":
            C.ckpt_window(ctx, True, T)  # let the remainder drain after the measured loop
        C.ckpt_wait(ctx, sid)
        snap_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    comp = [a.elapsed_time(b) for a, b, _ in evs]
    hbm = [b.elapsed_time(c) for _, b, c in evs]
    if ctx:
        C.ckpt_destroy(ctx)
    return {"iters": iters, "compute_ms": round(statistics.median(comp), 3),
            "hbm_ms": round(statistics.median(hbm), 3), "snapshot_s": round(snap_s, 3) if snap_s else None,
            "loop_ms": round(sum(comp) + sum(hbm), 1)}


res = {"none": run("none", 20), "ungated": run("ungated", 20), "gated": run("gated", 40),
       "none_again": run("none", 20)}
print(json.dumps(res))
