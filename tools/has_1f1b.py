#!/usr/bin/env python3
"""HAS (Alg 1, P.377-425) driven by a real 2-stage 1F1B pipeline on 2 GPUs.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
      tools/has_1f1b.py [--microbatches 8] [--layers 8] [--out profiles/r02/has_1f1b.jsonl]

Each rank is one pipeline stage p of |P| = 2 (Llama-2-13B TP4 x PP2, C3: rank p holds the
TP-rank-0 shard of stage p, 22.8 GB, snapshotted by its own context, m = 1).  One training
iteration on each stage:
  * 1F1B over M micro-batches (Megatron order: stage 0 runs one warm-up forward, then
    F(i+1) / B(i) pairs; stage 1 runs F(i) B(i)); a forward is `layers` bf16 GEMMs
    [tokens x h] @ [h x h], a backward twice that; activations / gradients cross NVLink
    with NCCL send/recv, batched in the steady state (send-forward + recv-backward);
  * a gradient all-reduce between the two stages (the tied-embedding all-reduce of
    pipeline parallelism; NCCL over NVLink) -- the communication phase;
  * an HBM-bound optimizer-like phase (fp32 axpy over 2 x 2 GiB).
The training stream opens HAS windows with stream memory operations (ckpt_window): BUBBLE
while it waits for a peer's activation/gradient, COMPUTE around the GEMM phases, COMM
around the all-reduce, and closes them for the optimizer phase.

Alg 1's inputs are MEASURED here: C_FB,BP = F + B of one micro-batch on this stage
(CUDA events), B_io = the ungated snapshot's host-link rate; EstimateBubbleTime /
SplitParameter come from ckpt_has_plan3 (Layer 2 capacity = the iteration's GEMM time,
reading Q28).  Placements, each snapshot issued at an iteration start while training runs
until it commits:
  ungated        -- every bucket's D2H runs whenever the copy engine gets to it;
  layer1         -- every bucket waits for a bubble;
  layers12       -- Alg 1's W_bubble in bubbles, the rest in compute (or bubble) windows;
  layers123      -- as layers12, and the W_comm tail also in communication windows.
Reported per placement (max over the two stages): iteration time while the snapshot is in
flight vs alone, per-phase times (optimizer phase, all-reduce) and the snapshot duration.
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--microbatches", type=int, default=8)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=8192)
    ap.add_argument("--allreduce-mib", type=int, default=1024)
    ap.add_argument("--opt-gib", type=int, default=2)
    ap.add_argument("--bucket-mib", type=int, default=32)
    ap.add_argument("--config", default="c3_13b_tp4pp2")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--out", default="")
    ap.add_argument("--watchdog-s", type=float, default=600.0)
    a = ap.parse_args()

    import faulthandler

    import torch
    import torch.distributed as dist

    from paper_2310_12670_b200 import ckpt as C
    from synth.gpu import descriptors, make_rank_state

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    if a.watchdog_s > 0:  # a hang dumps every thread's stack and exits instead of burning the call
        faulthandler.dump_traceback_later(a.watchdog_s, exit=True)
    t_start = time.time()

    def trace(*x):
        print(f"[has_1f1b rank {rank} +{time.time() - t_start:7.1f}s]", *x, file=sys.stderr, flush=True)

    assert world == 2, "a 2-stage pipeline: run on 2 GPUs"
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    p, P, peer = rank, world, 1 - rank
    M, h, T = a.microbatches, a.hidden, a.tokens

    # ---- model / training buffers --------------------------------------------------
    Ws = [torch.randn(h, h, dtype=torch.bfloat16, device=dev) * 0.01 for _ in range(a.layers)]
    x0 = torch.randn(T, h, dtype=torch.bfloat16, device=dev)
    act = [torch.empty(T, h, dtype=torch.bfloat16, device=dev) for _ in range(M)]
    grd = [torch.empty(T, h, dtype=torch.bfloat16, device=dev) for _ in range(M)]
    gbuf = torch.randn(a.allreduce_mib << 19, dtype=torch.bfloat16, device=dev)
    nopt = (a.opt_gib << 30) // 4
    master = torch.randn(nopt, dtype=torch.float32, device=dev)
    upd = torch.randn(nopt, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream()

    def fwd(i):
        x = x0 if p == 0 else act[i]
        for W in Ws:
            x = x @ W
        if p == 0:
            act[i].copy_(x)
        return x

    def bwd(i):
        g = grd[i]  # stage P-1: the loss gradient (synthetic); stage 0: received from stage 1
        y = x0 if p == 0 else act[i]
        for W in reversed(Ws):
            torch.matmul(g, W.t())   # dX
            torch.matmul(y.t(), g)   # dW
        return g

    ctx = None

    def window(mask):
        if ctx is not None:
            C.ckpt_window(ctx, mask, s)

    def wait_peer(works):
        window(C.CKPT_WINDOW_BUBBLE)  # the device idles until the peer's tensor arrives
        for w in works:
            w.wait()
        window(C.CKPT_WINDOW_COMPUTE)

    ev = {}

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        ev[name] = e

    def iteration():
        mark("t0")
        window(C.CKPT_WINDOW_COMPUTE)
        if p == 0:
            fwd(0)
            wait_peer([dist.isend(act[0], peer)])
            for i in range(M - 1):
                fwd(i + 1)
                wait_peer(dist.batch_isend_irecv([dist.P2POp(dist.isend, act[i + 1], peer),
                                                  dist.P2POp(dist.irecv, grd[i], peer)]))
                bwd(i)
            wait_peer([dist.irecv(grd[M - 1], peer)])
            bwd(M - 1)
        else:
            wait_peer([dist.irecv(act[0], peer)])
            for i in range(M - 1):
                fwd(i)
                bwd(i)
                wait_peer(dist.batch_isend_irecv([dist.P2POp(dist.isend, grd[i], peer),
                                                  dist.P2POp(dist.irecv, act[i + 1], peer)]))
            fwd(M - 1)
            bwd(M - 1)
            wait_peer([dist.isend(grd[M - 1], peer)])
        mark("pipe")
        window(C.CKPT_WINDOW_COMM)          # Layer 3: NVLink collective, the D2H is on PCIe
        dist.all_reduce(gbuf)
        mark("ar")
        window(0)                            # HBM-bound phase: every window closed
        master.add_(upd, alpha=1e-3)
        master.add_(upd, alpha=-1e-3)
        mark("opt")
        window(C.CKPT_WINDOW_COMPUTE)

    def timed_iteration():
        iteration()
        s.synchronize()
        return {"iter_ms": ev["t0"].elapsed_time(ev["opt"]), "pipe_ms": ev["t0"].elapsed_time(ev["pipe"]),
                "allreduce_ms": ev["pipe"].elapsed_time(ev["ar"]), "opt_ms": ev["ar"].elapsed_time(ev["opt"])}

    def allmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- C_FB,BP of this stage (one micro-batch, F + B, no communication) -------------
    for i in range(3):
        fwd(0)
        bwd(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(5):
        fwd(0)
        bwd(0)
    e1.record(s)
    e1.synchronize()
    c_fb_bp = e0.elapsed_time(e1) / 5 / 1e3
    trace(f"C_FB,BP = {c_fb_bp * 1e3:.2f} ms")
    for _ in range(3):
        timed_iteration()
    dist.barrier()
    base = [timed_iteration() for _ in range(8)]
    base_iter = statistics.median(x["iter_ms"] for x in base)
    trace(f"baseline iteration {base_iter:.2f} ms")

    # ---- snapshot state of this stage -----------------------------------------------
    specs, ts = make_rank_state(a.config, 4 * p, dev)
    S = sum(x.nbytes for x in specs)
    bucket = a.bucket_mib << 20
    results = {}

    def make_ctx(windowed):
        flags = C.CKPT_OPT_TIMING | (C.CKPT_OPT_WINDOWED if windowed else 0)
        c = C.ckpt_create(local, C.ckpt_options_default(n_slots=0, bucket_bytes=bucket, flags=flags, host_buffers=1))
        C.ckpt_register(c, descriptors(ts, specs))
        C.ckpt_protect(c, 1, 0)
        return c

    def run_placement(name, windowed, bubble_bytes, compute_bytes):
        nonlocal ctx
        ctx = make_ctx(windowed)
        C.ckpt_has_apply_layers(ctx, bubble_bytes, compute_bytes)
        window(C.CKPT_WINDOW_COMPUTE)
        out = []
        for rep in range(a.reps):
            dist.barrier()
            timed_iteration()
            t0 = time.perf_counter()
            sid = C.ckpt_snapshot(ctx, bucket, s)
            its = []
            done = False
            while not done:
                its.append(timed_iteration())
                done = C.ckpt_test(ctx, sid)
                flag = torch.tensor([0.0 if done else 1.0], device=dev)
                dist.all_reduce(flag)                # both stages keep training until both commit
                done = flag.item() == 0.0
                if len(its) > 400:
                    raise RuntimeError(f"{name}: snapshot did not complete in 400 iterations")
            C.ckpt_wait(ctx, sid)
            wall = time.perf_counter() - t0
            trace(f"{name} rep {rep}: committed after {len(its)} iterations, {wall:.2f} s")
            st = C.ckpt_get_stats(ctx)
            during = its[:-1] if len(its) > 1 else its  # the last iteration may end after the commit
            out.append({"iters": len(its),
                        "iter_ms": allmax(statistics.mean(x["iter_ms"] for x in during)),
                        "opt_ms": allmax(statistics.mean(x["opt_ms"] for x in during)),
                        "allreduce_ms": allmax(statistics.mean(x["allreduce_ms"] for x in during)),
                        "pipe_ms": allmax(statistics.mean(x["pipe_ms"] for x in during)),
                        "snapshot_ms": allmax(st["last_snapshot_ms"]), "wall_s": allmax(wall)})
        C.ckpt_destroy(ctx)
        ctx = None
        r = {k: statistics.median(x[k] for x in out) for k in out[0]}
        r["reps"] = out
        results[name] = r
        return r

    # ungated first: it gives B_io (the rate Alg 1's EstimateSnapshotTime assumes)
    ung = run_placement("ungated", False, 2 ** 64 - 1, 2 ** 64 - 1)
    b_io = S / (ung["snapshot_ms"] / 1e3)
    t_compute = statistics.median(x["pipe_ms"] for x in base) / 1e3 - 0.0  # GEMM phases of one iteration
    plan = C.ckpt_has_plan3(p, P, c_fb_bp, S, b_io, t_compute)
    trace("plan", plan)
    run_placement("layer1", True, 2 ** 64 - 1, 0)
    run_placement("layers12", True, plan["bubble_bytes"], 2 ** 64 - 1)
    run_placement("layers123", True, plan["bubble_bytes"], plan["compute_bytes"])

    base_m = {k: allmax(statistics.median(x[k] for x in base)) for k in base[0]}
    for name, r in results.items():
        r["iter_overhead_pct"] = round((r["iter_ms"] / base_m["iter_ms"] - 1) * 100, 3)
        r["opt_phase_overhead_pct"] = round((r["opt_ms"] / base_m["opt_ms"] - 1) * 100, 3)
        r["allreduce_overhead_pct"] = round((r["allreduce_ms"] / base_m["allreduce_ms"] - 1) * 100, 3)
    plans = [None, None]
    dist.all_gather_object(plans, {"stage": p, "c_fb_bp_ms": round(c_fb_bp * 1e3, 3), "b_io_gbs": round(b_io / 1e9, 2),
                                   "t_compute_ms": round(t_compute * 1e3, 2), **{k: (round(v, 4) if isinstance(v, float) else v)
                                                                                 for k, v in plan.items()}})
    if rank == 0:
        line = {"tool": "has_1f1b", "config": a.config, "state_bytes_per_stage": S, "stages": P, "microbatches": M,
                "layers_per_stage": a.layers, "gemm": f"[{T}x{h}]@[{h}x{h}] bf16", "allreduce_mib": a.allreduce_mib,
                "opt_phase_gib": 2 * a.opt_gib, "bucket_mib": a.bucket_mib, "baseline": base_m, "alg1_plan": plans,
                "placements": {k: {kk: (round(vv, 3) if isinstance(vv, float) else vv) for kk, vv in v.items()
                                   if kk != "reps"} for k, v in results.items()},
                "reps": {k: v["reps"] for k, v in results.items()}}
        txt = json.dumps(line)
        print(txt, flush=True)
        if a.out:
            with open(a.out, "a") as f:
                f.write(txt + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
