#!/usr/bin/env python3
"""Where does a snapshot's cost to a co-running GEMM come from?  (one GPU, C2 rank)

bf16 8192^3 GEMMs back to back on a high-priority stream; each window records every
GEMM's start/end.  Per kind, ABBA pairs of (alone, with) windows; the with-window starts
its traffic `--lead-ms` after the first GEMM, and we report the GEMMs overlapping the
traffic against (a) the same window's GEMMs after it ended and (b) the alone window:

  raw_d2h      pinned D2H of the 11.8 GB staging in 512 MiB copies (torch, no library)
  raw_d2h_poll the same with a host thread calling cudaStreamQuery every 200 us (ckpt_wait)
  lib_ce       ckpt_snapshot with the copy-engine pack (zero SMs) + ckpt_wait
  lib_kernel   ckpt_snapshot with the default TMA pack kernel + ckpt_wait
JSON line per kind on stderr, one summary line on stdout.
   python tools/corun_probe.py [--pairs 10] [--lead-ms 20]"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=10)
    ap.add_argument("--lead-ms", type=float, default=20.0)
    ap.add_argument("--kinds", default="raw_d2h,raw_d2h_poll,lib_ce,lib_kernel")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2310_12670_b200 import ckpt as C
    from synth.gpu import descriptors, make_rank_state
    dev = torch.device("cuda", 0)
    specs, ts = make_rank_state("c2_7b_tp8", 0, dev)
    S = sum(s.nbytes for s in specs)
    n = 8192
    A = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    Bm = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    hi = torch.cuda.Stream(device=dev, priority=-5)
    lo = torch.cuda.Stream(device=dev, priority=0)
    caller = torch.cuda.current_stream()
    stage = torch.empty(S, dtype=torch.uint8, device=dev)
    host = bench.registered_host_buffer(torch, S)
    P = 512 << 20

    def make(flags):
        ctx = C.ckpt_create(0, C.ckpt_options_default(n_slots=0, bucket_bytes=P, flags=C.CKPT_OPT_TIMING | flags))
        C.ckpt_register(ctx, descriptors(ts, specs))
        C.ckpt_protect(ctx, 1, 0)
        sid = C.ckpt_snapshot(ctx, P, caller)
        C.ckpt_wait(ctx, sid)
        return ctx

    ctxs = {"lib_ce": None, "lib_kernel": None}
    with torch.cuda.stream(hi):
        for _ in range(5):
            torch.matmul(A, Bm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(hi)
    with torch.cuda.stream(hi):
        for _ in range(20):
            torch.matmul(A, Bm)
    e1.record(hi)
    e1.synchronize()
    per = e0.elapsed_time(e1) / 20
    iters = int(3 * 240 / per)   # ~3x a snapshot
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]

    def window(kind):
        torch.cuda.synchronize()
        base = torch.cuda.Event(enable_timing=True)
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        base.record(hi)

        def gemms():  # enqueued from its own thread: a full launch queue must not delay the traffic
            with torch.cuda.stream(hi):
                for g0, g1 in ev:
                    g0.record(hi)
                    torch.matmul(A, Bm)
                    g1.record(hi)
        gt = threading.Thread(target=gemms)
        gt.start()
        stop = [False]
        poller = None
        if kind:
            time.sleep(a.lead_ms / 1e3)  # the GEMM stream is busy before the traffic starts
            if kind.startswith("raw"):
                t0e.record(lo)
                with torch.cuda.stream(lo):
                    for o in range(0, S - P + 1, P):
                        host.t[o:o + P].copy_(stage[o:o + P], non_blocking=True)
                t1e.record(lo)
                if kind == "raw_d2h_poll":
                    def poll():
                        while not stop[0]:
                            lo.query()
                            time.sleep(200e-6)
                    poller = threading.Thread(target=poll, daemon=True)
                    poller.start()
                t1e.synchronize()
            else:
                ctx = ctxs[kind]
                t0e.record(caller)
                sid = C.ckpt_snapshot(ctx, P, caller)
                C.ckpt_wait(ctx, sid)
                t1e.record(caller)
        gt.join()
        torch.cuda.synchronize()
        stop[0] = True
        if poller:
            poller.join()
        spans = [(base.elapsed_time(g0), base.elapsed_time(g1)) for g0, g1 in ev]
        tr = (base.elapsed_time(t0e), base.elapsed_time(t1e)) if kind else None
        return spans, tr

    out = {"tool": "corun_probe", "gemm_ms_each": round(per, 4), "iters": iters, "pairs": a.pairs, "lead_ms": a.lead_ms}
    for kind in a.kinds.split(","):
        if kind in ctxs:
            for k, c in ctxs.items():
                if c is not None:
                    C.ckpt_destroy(c)
                    ctxs[k] = None
            ctxs[kind] = make(C.CKPT_OPT_CE_PACK if kind == "lib_ce" else 0)
        rows = []
        for i in range(a.pairs):
            order = (None, kind) if i % 2 == 0 else (kind, None)
            res = {k: window(k) for k in order}
            alone = [b - a_ for a_, b in res[None][0][2:]]
            spans, (ta, tb) = res[kind]
            during = [b - a_ for a_, b in spans if a_ >= ta and b <= tb]
            after = [b - a_ for a_, b in spans if a_ > tb + 1.0]
            ma, md, mf = statistics.mean(alone), statistics.mean(during), statistics.mean(after) if after else None
            rows.append({"during_vs_after": (md / mf - 1) * 100 if mf else None, "during_vs_alone": (md / ma - 1) * 100,
                         "after_vs_alone": (mf / ma - 1) * 100 if mf else None, "traffic_ms": tb - ta,
                         "n_during": len(during), "n_after": len(after)})
        summ = {k: round(statistics.median(r[k] for r in rows if r[k] is not None), 3)
                for k in ("during_vs_after", "during_vs_alone", "after_vs_alone", "traffic_ms", "n_during", "n_after")}
        summ["spread_during_vs_alone"] = round(max(r["during_vs_alone"] for r in rows) - min(r["during_vs_alone"] for r in rows), 3)
        out[kind] = summ
        print(json.dumps({kind: summ}), file=sys.stderr, flush=True)
    for c in ctxs.values():
        if c is not None:
            C.ckpt_destroy(c)
    host.release()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
