#!/usr/bin/env python3
"""Failure drill under torchrun's elastic agent (REFT-load, P.545, P.551-555; SPEC S.514).

  python -m torch.distributed.run --nnodes 1 --nproc-per-node N --max-restarts 1 \
      --master-addr 127.0.0.1 --master-port P tools/elastic_drill.py --key K --out DIR

Attempt 0 (TORCHELASTIC_RESTART_COUNT = 0): every rank registers a seeded state, protects
it in one AEC group over CUDA IPC with a persistent shared-memory arena (arena_key K),
commits two snapshots (v1, then v2 after mutating the tensors), then rank N-1 loses its
host memory (its arena files are removed) and its process dies (os._exit).  The agent sees
the failure, stops the other workers and starts a NEW process per GPU.

Attempt 1: each new process re-creates its context with the same key: the survivors
re-attach their committed v2 host images, the replaced rank finds none; the group
protects again (the committed version is v2), ckpt_recover rebuilds the replaced member
from the survivors' images and parity (Eq 2), every rank loads, and every byte of every
tensor is compared with the generator's v2 bytes.  Each rank writes DIR/rank<r>.json.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--key", type=lambda x: int(x, 0), required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--config", default="tiny_7")
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2310_12670_b200 import ckpt as C
    from synth.gpu import alloc_state, descriptors, fill_state

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    attempt = int(os.environ.get("TORCHELASTIC_RESTART_COUNT", "0"))
    lost = world - 1
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # torchrun's static rendezvous (--master-addr/--master-port) keeps ONE agent store across
    # restarts and gives the workers no per-attempt prefix, so a restarted group would read
    # attempt 0's NCCL bootstrap keys (a dead rank 0's address): prefix them by attempt
    from datetime import timedelta
    agent_store = os.environ.get("TORCHELASTIC_USE_AGENT_STORE") == "True"
    base = dist.TCPStore(os.environ["MASTER_ADDR"], int(os.environ["MASTER_PORT"]), world,
                         is_master=(not agent_store and rank == 0), timeout=timedelta(seconds=300))
    store = dist.PrefixStore(f"/reft-elastic-drill/attempt{attempt}", base)
    dist.init_process_group("nccl", store=store, rank=rank, world_size=world, device_id=dev)
    specs = synth.config_tensors(a.config, rank)
    ts = alloc_state(specs, dev, misalign=1)
    o = C.ckpt_options_default(n_slots=0, bucket_bytes=1 << 16, stripe_unit=4096, flags=C.CKPT_OPT_SHM_ARENA,
                               arena_key=a.key)
    ctx = C.ckpt_create(local, o)
    C.ckpt_register(ctx, descriptors(ts, specs), {"rank": rank, "world": world, "local_rank": local,
                                                  "local_world": world})
    C.protect_ipc(ctx)
    if attempt == 0:
        fill_state(ts, rank)
        sid = C.ckpt_snapshot(ctx)
        C.ckpt_wait(ctx, sid)                       # v1
        fill_state(ts, rank, seed=31, xor_mode=1)   # a later training step
        sid = C.ckpt_snapshot(ctx)
        C.ckpt_wait(ctx, sid)                       # v2 = generator(SEED) ^ generator(31)
        dist.barrier()
        if rank == lost:                            # the node's memory goes with the process
            for b in range(2):
                try:
                    os.unlink(f"/dev/shm/reft-{a.key:016x}-{rank}-{b}")
                except FileNotFoundError:
                    pass
            os._exit(13)
        dist.barrier()                              # never passes: the agent restarts the group
        raise SystemExit("unreachable: the lost rank did not die")
    for t in ts:
        t.view(torch.uint8).fill_(0x77)             # a fresh process: garbage in the tensors
    g = C.ckpt_geometry(ctx)
    C.ckpt_recover(ctx, 1 << lost)
    C.ckpt_load(ctx)
    torch.cuda.synchronize()
    bad = []
    for t, x in enumerate(ts):
        want = synth.fill(synth.SEED, rank, t, specs[t].nbytes) ^ synth.fill(31, rank, t, specs[t].nbytes)
        if not np.array_equal(x.contiguous().view(torch.uint8).cpu().numpy(), want):
            bad.append(t)
    C.ckpt_destroy(ctx)
    dist.barrier()
    dist.destroy_process_group()
    with open(os.path.join(a.out, f"rank{rank}.json"), "w") as f:
        json.dump({"rank": rank, "attempt": attempt, "lost": lost, "m": g["m"], "tensors": len(specs),
                   "bad_tensors": bad, "ok": not bad}, f)


if __name__ == "__main__":
    try:
        main()
    except BaseException:  # the agent reports only exit codes: keep each attempt's traceback
        import traceback
        d = sys.argv[sys.argv.index("--out") + 1]
        with open(os.path.join(d, f"rank{os.environ.get('RANK')}_attempt{os.environ.get('TORCHELASTIC_RESTART_COUNT')}.err"), "w") as f:
            f.write(traceback.format_exc())
        raise
