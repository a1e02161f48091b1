#!/usr/bin/env python3
"""One process, m GPUs: a CKPT_GROUP_LOCAL group whose members sit on different devices,
so the XOR encode reads its peers over NVLink inside a single process -- the only way to
put the NVLink-bound kernel under ncu (never a multi-rank command).

  python tools/xor_local2.py [--m 2] [--config c2_7b_tp8] [--reps 3] [--device-only]

Prints per-kernel mean launch times and NVLink GB/s (CUDA events on the launch stream)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--m", type=int, default=2)
    p.add_argument("--config", default="c2_7b_tp8")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--bucket", type=int, default=64 << 20)
    p.add_argument("--flags", type=int, default=0)
    p.add_argument("--unit", type=int, default=1 << 20, help="stripe unit u (Q4)")
    p.add_argument("--with-d2h", action="store_true", help="run a pinned D2H on every device meanwhile")
    p.add_argument("--rebuild", type=int, default=-1,
                   help="then lose member k (device copy + host image) and rebuild it from the survivors' "
                        "device images (Eq 2): rebuild kernel per launch, bytes and GB/s")
    a = p.parse_args()
    import torch

    from paper_2310_12670_b200 import ckpt as C
    from synth.gpu import descriptors, make_rank_state

    m = min(a.m, torch.cuda.device_count())
    ctxs, states = [], []
    for j in range(m):
        torch.cuda.set_device(j)
        specs, ts = make_rank_state(a.config, j, torch.device("cuda", j))
        c = C.ckpt_create(j, C.ckpt_options_default(n_slots=0, bucket_bytes=a.bucket, stripe_unit=a.unit,
                                                    flags=C.CKPT_OPT_TIMING | C.CKPT_OPT_DEVICE_ONLY | a.flags))
        C.ckpt_register(c, descriptors(ts, specs))
        ctxs.append(c)
        states.append((specs, ts))
    C.protect_local(ctxs)
    side, hbs, dbs = [], [], []
    if a.with_d2h:
        for j in range(m):
            side.append(torch.cuda.Stream(device=j))
            hbs.append(torch.empty(4 << 30, dtype=torch.uint8, pin_memory=True))
            dbs.append(torch.empty(4 << 30, dtype=torch.uint8, device=f"cuda:{j}"))
    for r in range(a.reps + 1):
        for j in range(len(side)):
            with torch.cuda.stream(side[j]):
                hbs[j].copy_(dbs[j], non_blocking=True)
        if r == 1:
            for c in ctxs:
                C.ckpt_stats_reset(c)
        ids = []
        for j, c in enumerate(ctxs):
            torch.cuda.set_device(j)
            ids.append(C.ckpt_snapshot(c, 0, torch.cuda.current_stream(j)))
        for c, i in zip(ctxs, ids):
            C.ckpt_wait(c, i)
    st = C.ckpt_get_stats(ctxs[0])
    print(json.dumps({"m": m, "config": a.config, "unit": C.ckpt_geometry(ctxs[0])["unit"], "pack_us": st["pack_ms"] / max(st["pack_launches"], 1) * 1e3,
                      "xor_us": st["xor_ms"] / max(st["xor_launches"], 1) * 1e3,
                      "xor_nvlink_gbs": st["xor_bytes_in"] / max(st["xor_ms"], 1e-9) / 1e6,
                      "pack_hbm_gbs": st["pack_bytes"] / max(st["pack_ms"], 1e-9) / 1e6,
                      "snapshot_ms": st["last_snapshot_ms"],
                      # m = 2 + CKPT_OPT_CE_GATHER: the copy-engine mirror (no XOR kernel)
                      "ce_mirror_ms": st["gather_ms"] / a.reps if st["gather_ops"] else None,
                      "ce_mirror_nvlink_gbs": C.ckpt_geometry(ctxs[0])["L_star"] * a.reps / st["gather_ms"] / 1e6
                      if st["gather_ops"] and st["gather_ms"] > 0 else None}))
    if a.rebuild >= 0:
        k = a.rebuild
        g = C.ckpt_geometry(ctxs[0])
        for rep in range(2):
            for c in ctxs:
                C.ckpt_stats_reset(c)
            C.ckpt_forget(ctxs[k], 0xA5)
            torch.cuda.set_device(k)
            for t in states[k][1]:
                t.view(torch.uint8).fill_(0xA5)  # the lost member's tensors are gone too
            for j, c in enumerate(ctxs):
                torch.cuda.set_device(j)
                C.ckpt_rebuild(c, k, torch.cuda.current_stream(j))
            for j in range(m):
                torch.cuda.synchronize(j)
        rows = []
        for j, c in enumerate(ctxs):
            st = C.ckpt_get_stats(c)
            if st["rebuild_launches"]:
                rows.append({"member": j, "launches": st["rebuild_launches"],
                             "kernel_us": round(st["rebuild_ms"] / st["rebuild_launches"] * 1e3, 2),
                             "bytes_in": st["rebuild_bytes_in"], "bytes_out": st["rebuild_bytes_out"],
                             "gbs_in_plus_out": round((st["rebuild_bytes_in"] + st["rebuild_bytes_out"])
                                                      / max(st["rebuild_ms"], 1e-9) / 1e6, 1)})
        # bit-exact: the lost member's tensors after a load equal the generator
        from synth import SEED, fill as gfill
        C.ckpt_load(ctxs[k], torch.cuda.current_stream(k))
        torch.cuda.synchronize(k)
        specs, ts = states[k]
        ok = all(bool((ts[t].view(torch.uint8).cpu().numpy()[:4096] ==
                       gfill(SEED, k, t, min(4096, specs[t].nbytes))).all()) for t in range(0, len(ts), 37))
        print(json.dumps({"rebuild_lost": k, "m": m, "L_star": g["L_star"], "row_owners": rows, "sampled_ok": ok}))
    for c in ctxs:
        C.ckpt_destroy(c)


if __name__ == "__main__":
    main()
