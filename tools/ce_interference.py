#!/usr/bin/env python3
"""Does copy-engine traffic slow the pack kernel?  Device-only single-launch pack of the
C2 state (no D2H of its own), alone and while another stream runs pinned D2H / H2D /
D2D copies (one big copy or 64 MiB pieces), for two bucket sizes.  Prints the mean
pack-kernel time per condition (CUDA events, CKPT_OPT_TIMING)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2310_12670_b200 import ckpt as C  # noqa: E402
from synth.gpu import descriptors, make_rank_state  # noqa: E402

specs, ts = make_rank_state("c2_7b_tp8", 0, "cuda:0")
side = torch.cuda.Stream()
hb = torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True)
db = torch.empty(4 << 30, dtype=torch.uint8, device="cuda:0")
db2 = torch.empty(4 << 30, dtype=torch.uint8, device="cuda:0")
res = {}
for bucket in (64 << 20, 256 << 20):
    ctx = C.ckpt_create(0, C.ckpt_options_default(n_slots=0, bucket_bytes=bucket,
                                                  flags=C.CKPT_OPT_TIMING | C.CKPT_OPT_DEVICE_ONLY))
    C.ckpt_register(ctx, descriptors(ts, specs))
    C.ckpt_protect(ctx, 1, 0)
    for cond in ["alone", "d2h_big", "d2h_64m", "h2d_big", "d2d_big"]:
        for rep in range(4):
            if rep == 1:
                C.ckpt_stats_reset(ctx)
            torch.cuda.synchronize()
            with torch.cuda.stream(side):
                if cond == "d2h_big":
                    hb.copy_(db, non_blocking=True)
                elif cond == "d2h_64m":
                    for i in range(64):
                        hb[i << 26:(i + 1) << 26].copy_(db[i << 26:(i + 1) << 26], non_blocking=True)
                elif cond == "h2d_big":
                    db.copy_(hb, non_blocking=True)
                elif cond == "d2d_big":
                    db2.copy_(db, non_blocking=True)
            sid = C.ckpt_snapshot(ctx)
            C.ckpt_wait(ctx, sid)
        torch.cuda.synchronize()
        st = C.ckpt_get_stats(ctx)
        ms = st["pack_ms"] / st["pack_launches"]
        res[f"B{bucket >> 20}M_{cond}"] = {"pack_ms": round(ms, 3),
                                           "pack_gbs": round(st["pack_bytes"] / st["pack_launches"] / ms / 1e6, 1)}
    C.ckpt_destroy(ctx)
print(json.dumps(res))
