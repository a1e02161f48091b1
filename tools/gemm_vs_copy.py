#!/usr/bin/env python3
"""What in a snapshot slows a co-running GEMM?  bf16 8192^3 GEMMs back to back on a
high-priority stream (bench.py's co-run GEMM) while a least-priority side stream runs one
kind of copy-engine traffic for the whole window, no library involved:

  d2h       pinned D2H of a 4 GiB device buffer in 512 MiB copies (the snapshot's D2H)
  d2h_l2    the same copies from a 64 MiB source (L2-resident: no HBM reads)
  h2d       pinned H2D into a 4 GiB device buffer in 512 MiB copies (PCIe the other way)
  d2d_paced device-to-device 512 MiB copies issued every ~9 ms by the host (~55 GB/s of
            HBM read + write, like the D2H's rate, without PCIe; no sleep kernel)

Per kind: 8 pairs of GEMM windows (alone / with traffic, ABBA order), whole-window slowdown
median/min/max, the side stream's GB/s, and the NVML SM clock / power of both windows.
One JSON line.   python tools/gemm_vs_copy.py [--pairs 8] [--iters 300]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=8)
    ap.add_argument("--iters", type=int, default=300)
    a = ap.parse_args()
    import torch

    import bench
    dev = torch.device("cuda", 0)
    n = 8192
    A = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    Bm = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    hi = torch.cuda.Stream(device=dev, priority=-5)
    lo = torch.cuda.Stream(device=dev, priority=0)
    big = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    big2 = torch.empty(4 << 30, dtype=torch.uint8, device=dev)
    small = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    host = bench.registered_host_buffer(torch, 4 << 30)
    nvml = bench.NvmlSampler(torch, dev)
    P = 512 << 20

    def side(kind, stop_evt):
        """Enqueue traffic on `lo` until roughly the GEMM window's length; returns bytes."""
        moved = 0
        with torch.cuda.stream(lo):
            for r in range(400):
                for o in range(0, 4 << 30, P):
                    if kind == "d2h":
                        host.t[o:o + P].copy_(big[o:o + P], non_blocking=True)
                    elif kind == "d2h_l2":
                        for q in range(0, P, 64 << 20):
                            host.t[o + q:o + q + (64 << 20)].copy_(small, non_blocking=True)
                    elif kind == "h2d":
                        big[o:o + P].copy_(host.t[o:o + P], non_blocking=True)
                    moved += P
                    if moved >= stop_evt:
                        return moved
        return moved

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
    per_ms = e0.elapsed_time(e1) / 20
    win_ms = per_ms * a.iters

    def window(kind):
        torch.cuda.synchronize()
        nvml.start()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        moved = 0
        if kind and kind != "d2d_paced":
            s0.record(lo)
            # enough traffic for the window at the host link's ~55 GB/s
            moved = side(kind, int(win_ms / 1e3 * 60e9))
            s1.record(lo)
        g0.record(hi)
        with torch.cuda.stream(hi):
            for _ in range(a.iters):
                torch.matmul(A, Bm)
        g1.record(hi)
        if kind == "d2d_paced":  # the host paces: one 512 MiB D2D copy every ~9 ms
            import time
            s0.record(lo)
            o = 0
            while not g1.query():
                with torch.cuda.stream(lo):
                    big2[o:o + P].copy_(big[o:o + P], non_blocking=True)
                moved += P
                o = (o + P) % (4 << 30)
                time.sleep(0.009)
            s1.record(lo)
        torch.cuda.synchronize()
        c = nvml.stop()
        gbs = moved / s0.elapsed_time(s1) / 1e6 if kind else None
        return g0.elapsed_time(g1), gbs, c

    out = {"tool": "gemm_vs_copy", "gemm": "bf16 8192^3 on a high-priority stream", "gemm_ms_each": round(per_ms, 4),
           "iters": a.iters, "pairs": a.pairs}
    for kind in ("d2h", "d2h_l2", "h2d", "d2d_paced"):
        rows = []
        for i in range(a.pairs):
            if i % 2 == 0:
                ta, _, ca = window(None)
                tw, gbs, cw = window(kind)
            else:
                tw, gbs, cw = window(kind)
                ta, _, ca = window(None)
            rows.append({"slow_pct": (tw / ta - 1) * 100, "side_gbs": gbs,
                         "mhz_alone": ca and ca["sm_mhz"], "mhz_with": cw and cw["sm_mhz"],
                         "w_alone": ca and ca["power_w"], "w_with": cw and cw["power_w"]})
        med = lambda k: round(statistics.median(r[k] for r in rows if r[k] is not None), 3) if any(r[k] is not None for r in rows) else None
        out[kind] = {"slowdown_pct": med("slow_pct"), "min": round(min(r["slow_pct"] for r in rows), 3),
                     "max": round(max(r["slow_pct"] for r in rows), 3), "side_gbs": med("side_gbs"),
                     "sm_mhz_alone": med("mhz_alone"), "sm_mhz_with": med("mhz_with"),
                     "power_w_alone": med("w_alone"), "power_w_with": med("w_with")}
        print(json.dumps({kind: out[kind]}), file=sys.stderr, flush=True)
    host.release()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
