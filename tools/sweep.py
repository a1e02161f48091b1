#!/usr/bin/env python3
"""Per-config measurements for SURVEY.md 8(d) (C1-C5), one process per GPU.

  torchrun --nproc-per-node N tools/sweep.py --config c3_13b_tp4pp2 --buckets 4,16,64,256,512 --drill
  python tools/sweep.py --config c2_7b_tp8            (N = 1)

For every bucket size (MiB): snapshot+protect time (median of reps, max over ranks),
state GB/s per GPU, wire GB/s, device-side protect (DEVICE_ONLY) time, and with --drill
the rebuild of lost rank k plus the distributed in-memory load (C5), with a bit-exact
check of the rebuilt rank's tensors against the generator.  JSON lines on rank 0."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2_7b_tp8")
    p.add_argument("--buckets", default="64")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--n-slots", type=int, default=4)
    p.add_argument("--unit", type=int, default=1 << 20)
    p.add_argument("--flags", type=int, default=0)
    p.add_argument("--drill", action="store_true")
    p.add_argument("--device-only", action="store_true")
    p.add_argument("--lost", default="")
    p.add_argument("--scheme", type=int, default=0, help="CKPT_SCHEME_*: 1 AEC, 2 ARC, 3 ARC+AEC")
    p.add_argument("--host-buffers", type=int, default=2)
    p.add_argument("--corun", action="store_true", help="bf16 GEMM co-run slowdown per bucket size (bench.py's)")
    p.add_argument("--corun-pairs", type=int, default=12)
    p.add_argument("--max-ctas", default="0",
                   help="comma list of CTA budgets of the pack/XOR launches (0 = 2 x SMs); one record per budget")
    a = p.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2310_12670_b200 import ckpt as C
    from synth.gpu import descriptors, fill_state, make_rank_state

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

    specs, ts = make_rank_state(a.config, rank, dev)
    S = sum(s.nbytes for s in specs)
    for bmib, mc in [(int(x), int(y)) for x in a.buckets.split(",") for y in a.max_ctas.split(",")]:
        flags = a.flags | C.CKPT_OPT_TIMING | (C.CKPT_OPT_DEVICE_ONLY if a.device_only else 0)
        if a.scheme in (2, 3):
            flags |= C.CKPT_OPT_SHM_ARENA
        n_slots = 0 if a.device_only else a.n_slots
        ctx = C.ckpt_create(local, C.ckpt_options_default(bucket_bytes=bmib << 20, n_slots=n_slots,
                                                          stripe_unit=a.unit, flags=flags, max_ctas=mc,
                                                          host_buffers=a.host_buffers))
        C.ckpt_register(ctx, descriptors(ts, specs))
        if world > 1:
            C.protect_ipc(ctx, scheme=a.scheme)
        else:
            C.ckpt_protect(ctx, 1, 0)
        g = C.ckpt_geometry(ctx)
        st0 = torch.cuda.current_stream()
        times = []
        for r in range(a.reps + 1):
            bar()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sid = C.ckpt_snapshot(ctx, 0, st0)
            C.ckpt_wait(ctx, sid)
            dt = amax(time.perf_counter() - t0)
            if r:
                times.append(dt)
            else:
                C.ckpt_stats_reset(ctx)  # the first snapshot pays first-touch of peer mappings
        st = C.ckpt_get_stats(ctx)
        t = statistics.median(times)
        rec = {"config": a.config, "m": g["m"], "bucket_mib": bmib, "n_slots": n_slots, "flags": flags,
               "max_ctas": mc or "2 x SMs",
               "state_bytes": S, "L_star": g["L_star"], "snapshot_ms": round(t * 1e3, 3),
               "state_gbs_per_gpu": round(S / t / 1e9, 3), "wire_gbs_per_gpu": round(st["d2h_bytes"] / a.reps / t / 1e9, 3),
               "pack_us_per_launch": round(st["pack_ms"] / max(st["pack_launches"], 1) * 1e3, 2),
               "xor_us_per_launch": round(st["xor_ms"] / max(st["xor_launches"], 1) * 1e3, 2),
               "pack_hbm_gbs": round(st["pack_bytes"] / st["pack_ms"] / 1e6, 1) if st["pack_ms"] > 0 else None,
               "xor_nvlink_gbs": round(st["xor_bytes_in"] / st["xor_ms"] / 1e6, 1)
               if st["xor_ms"] > 0 and not (a.flags & C.CKPT_OPT_CE_GATHER) else None,
               "launches_per_snapshot": (st["pack_launches"] + st["xor_launches"]) // a.reps}
        if a.corun:
            import bench
            co = bench.gemm_corun(torch, C, ctx, st0, bmib << 20, bar, amax, dev, a.corun_pairs)
            rec["gemm_slowdown_pct"] = co["slowdown_pct"]
            rec["gemm_corun"] = {k: co[k] for k in ("whole_window", "in_window", "pack_window", "protect_window",
                                                    "snapshot_window", "clock_drop_pct", "sm_mhz", "power_w")}
        if a.drill and g["m"] >= 2:
            lost = [tuple(int(y) for y in x.split("+")) for x in a.lost.split(",")] if a.lost else [(0,), (g["m"] - 1,)]
            C.ckpt_stats_reset(ctx)
            for k in lost:
                mask = sum(1 << x for x in k)
                fill_state(ts, rank, seed=999 + mask, xor_mode=1)  # later steps mutate everything
                if rank in k:
                    C.ckpt_forget(ctx, 0xA5)
                    for x in ts:
                        x.view(torch.uint8).fill_(0xA5)
                bar()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                C.ckpt_recover(ctx, mask)
                t1 = time.perf_counter()
                h2d0 = C.ckpt_get_stats(ctx)["h2d_bytes"]
                C.ckpt_load(ctx, st0)
                st0.synchronize()  # the training stream is ready (a background host restore may continue)
                t2 = time.perf_counter()
                C.ckpt_sync(ctx)
                t3 = time.perf_counter()
                rb, ld, hs = amax(t1 - t0), amax(t2 - t1), amax(t3 - t0)
                per = [t2 - t1, float(C.ckpt_get_stats(ctx)["h2d_bytes"] - h2d0)]
                if world > 1:
                    g_ = [torch.zeros(2, dtype=torch.float64, device=dev) for _ in range(world)]
                    dist.all_gather(g_, torch.tensor(per, dtype=torch.float64, device=dev))
                    per_rank = [(round(x[0].item() * 1e3, 1), int(x[1].item())) for x in g_]
                else:
                    per_rank = [(round(per[0] * 1e3, 1), int(per[1]))]
                srb = C.ckpt_get_stats(ctx)
                # bit-exact, unsampled: every byte of every tensor of every rank equals the
                # generator's (regenerated on the device by the harness generator, which the
                # CPU tests pin to the oracle's copy and to the published SplitMix64 outputs)
                ok = True
                from synth import SEED
                scratch = torch.empty(max(s_.nbytes for s_ in specs), dtype=torch.uint8, device=dev)
                for ti, x in enumerate(ts):
                    n = specs[ti].nbytes
                    C.reft_synth_fill(scratch.data_ptr(), n, SEED, rank, ti, 0, None)
                    ok = ok and bool(torch.equal(x.contiguous().view(torch.uint8).reshape(-1), scratch[:n]))
                del scratch
                okall = amax(0.0 if ok else 1.0) == 0.0
                # rebuild kernel of this rank (a row owner), per launch: NVLink/HBM bytes in +
                # bytes stored into the lost rank over NVLink, / mean launch time
                kgbs = (srb["rebuild_bytes_in"] + srb["rebuild_bytes_out"]) / max(srb["rebuild_ms"], 1e-9) / 1e6
                rec.setdefault("drill", []).append({"lost": k, "rebuild_ms": round(rb * 1e3, 2), "load_ms": round(ld * 1e3, 2),
                                                    "host_reprotected_ms": round(hs * 1e3, 2),
                                                    "load_ms_h2d_bytes_per_rank": per_rank,
                                                    "bit_exact_all_bytes": okall,
                                                    "rank0_rebuild_kernel_gbs": round(kgbs, 1) if rank not in k else None,
                                                    "rank0_rebuild_launches": srb["rebuild_launches"]})
                C.ckpt_stats_reset(ctx)
        if rank == 0:
            print(json.dumps(rec), flush=True)
        C.ckpt_destroy(ctx)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
