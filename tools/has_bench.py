#!/usr/bin/env python3
"""HAS placement on B200 (Alg 1, P.377-429), N=1: a training-like loop of one pipeline stage
alternates a bubble (the GPU idles for EstimateBubbleTime of a 1F1B schedule, emulated with
a device-side sleep), a compute-bound phase (bf16 GEMMs) and an HBM-bound phase (an
Adam-like streaming update); a C2 snapshot runs meanwhile
  ungated : D2H whenever the copy engine gets to it,
  gated   : D2H only in the compute phases (ckpt_window, CKPT_OPT_WINDOWED),
  alg1    : Alg 1 -- ckpt_has_plan(stage, stages, C_FB,BP, bytes, B_io) splits the image,
            ckpt_has_apply places the first W_bubble bytes in the bubbles and the rest in
            the compute phases; the HBM phases stay closed.
Reports each phase's median time per mode and the snapshot's duration."""
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


BUBBLE_CYCLES = 0  # set from the measured compute phase (see below)
BUCKET = int(os.environ.get("HAS_BUCKET_MIB", "32")) << 20  # a window closes within ~1 bucket of D2H


def iteration(ctx, mode, evs):
    gated = mode in ("gated", "alg1")
    with torch.cuda.stream(T):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        if BUBBLE_CYCLES:
            if mode == "alg1":
                C.ckpt_window(ctx, C.CKPT_WINDOW_BUBBLE, T)
            torch.cuda._sleep(BUBBLE_CYCLES)  # the pipeline bubble: the GPU waits for a peer stage
        if gated:
            C.ckpt_window(ctx, C.CKPT_WINDOW_COMPUTE if mode == "alg1" else True, T)
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


def run(mode, iters, plan=None):
    """Median phase times over `iters` iterations issued right after the snapshot starts
    (sized so the snapshot is in flight for all of them)."""
    ctx = None
    if mode != "none":
        flags = C.CKPT_OPT_TIMING | (C.CKPT_OPT_WINDOWED if mode in ("gated", "alg1") else 0)
        ctx = C.ckpt_create(0, C.ckpt_options_default(n_slots=0, bucket_bytes=BUCKET, flags=flags))
        C.ckpt_register(ctx, descriptors(ts, specs))
        C.ckpt_protect(ctx, 1, 0)
        if plan is not None:
            C.ckpt_has_apply(ctx, plan["bubble_bytes"])
        sid = C.ckpt_snapshot(ctx, 0, T)  # warm-up snapshot (windows open)
        C.ckpt_wait(ctx, sid)
    for _ in range(3):
        iteration(ctx, "none", [])
    torch.cuda.synchronize()
    evs = []
    t0 = time.perf_counter()
    sid = C.ckpt_snapshot(ctx, 0, T) if ctx else None
    for i in range(iters):
        iteration(ctx, mode, evs)
    snap_s = None
    if ctx:
        if mode in ("gated", "alg1"):
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


# Alg 1's inputs, measured: C_FB,BP = one compute phase; B_io = the ungated snapshot rate.
base = run("none", 10)
c_fb = base["compute_ms"] / 1e3
stage, stages = 0, 2                      # first stage of a 2-stage 1F1B pipeline
probe = run("ungated", 20)
S = sum(sp.nbytes for sp in specs)
b_io = S / probe["snapshot_s"]
plan = C.ckpt_has_plan(stage, stages, c_fb, S, b_io)
per_iter_bubble = (0.8 * stage + 2 * stages - stage - 2) * c_fb   # EstimateBubbleTime, per iteration
BUBBLE_CYCLES = int(per_iter_bubble * 1.965e9)                    # sleep at the max SM clock
res = {"alg1_inputs": {"c_fb_bp_s": round(c_fb, 5), "stage": stage, "stages": stages, "snapshot_bytes": S,
                       "b_io_gbs": round(b_io / 1e9, 2), "bubble_ms_per_iter": round(per_iter_bubble * 1e3, 3),
                       "plan": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in plan.items()}},
       "none": run("none", 20), "ungated": run("ungated", 20), "gated": run("gated", 40),
       "alg1": run("alg1", 40, plan), "none_again": run("none", 20)}
print(json.dumps(res))
