#!/usr/bin/env python3
"""REFT-load (a8) on one GPU: ckpt_load from the device copy of the completed image (one
unpack launch) and from host (H2D + unpack), C2 7B/TP8 rank; unpack kernel GB/s from the
library's CUDA-event timing (2 x L HBM bytes per load) and the load's host wall time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2310_12670_b200 import ckpt as C  # noqa: E402
from synth.gpu import descriptors, make_rank_state  # noqa: E402

dev = torch.device("cuda", 0)
specs, ts = make_rank_state(os.environ.get("CONFIG", "c2_7b_tp8"), 0, dev)
out = {}
for name, flags in (("device", 0), ("host", C.CKPT_OPT_HOST_LOAD)):
    ctx = C.ckpt_create(0, C.ckpt_options_default(n_slots=0, bucket_bytes=512 << 20,
                                                  flags=C.CKPT_OPT_TIMING | flags))
    C.ckpt_register(ctx, descriptors(ts, specs))
    C.ckpt_protect(ctx, 1, 0)
    sid = C.ckpt_snapshot(ctx)
    C.ckpt_wait(ctx, sid)
    L = C.ckpt_geometry(ctx)["L"]
    C.ckpt_load(ctx)
    torch.cuda.synchronize()
    C.ckpt_stats_reset(ctx)
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        C.ckpt_load(ctx)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    st = C.ckpt_get_stats(ctx)
    per_ms = st["unpack_ms"] / max(st["unpack_launches"], 1)
    out[name] = {"load_ms_median": round(sorted(times)[2] * 1e3, 2), "unpack_launches_per_load": st["unpack_launches"] // 5,
                 "unpack_ms_per_load": round(st["unpack_ms"] / 5, 3),
                 "unpack_hbm_gbs": round(2 * L * 5 / (st["unpack_ms"] / 1e3) / 1e9, 1) if st["unpack_ms"] else None,
                 "h2d_gbs": round(st["h2d_bytes"] / 5 / (sorted(times)[2]) / 1e9, 2) if st["h2d_bytes"] else None}
    C.ckpt_destroy(ctx)
out["L"] = L
print(json.dumps(out))
