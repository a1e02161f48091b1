"""Multi-GPU parity of the IPC transport: one process per GPU (torch.distributed over
NCCL for the handle exchange only), peer slots mapped with CUDA IPC, per-bucket
ordering by stream memory operations, XOR parity read over NVLink.  Bit-exact vs the
oracle; rebuild drill for every lost rank.  Needs >= 2 GPUs (skipped otherwise)."""
import os
import socket
import traceback

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch
        import torch.distributed as dist

        import oracle
        import synth
        from paper_2310_12670_b200 import ckpt as C
        from synth.gpu import descriptors, fill_state, make_rank_state

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", device_id=dev)
        config, unit, n_slots, bucket, flags, misalign = case
        specs, ts = make_rank_state(config, rank, dev, misalign=misalign)
        ctx = C.ckpt_create(rank, C.ckpt_options_default(stripe_unit=unit, n_slots=n_slots, bucket_bytes=bucket,
                                                         flags=flags))
        C.ckpt_register(ctx, descriptors(ts, specs))
        C.protect_ipc(ctx)
        g = C.ckpt_geometry(ctx)
        sid = C.ckpt_snapshot(ctx)
        C.ckpt_wait(ctx, sid)
        # expected images of every rank from the oracle (deterministic generator)
        imgs = []
        for j in range(world):
            sp = synth.config_tensors(config, j)
            tb = [synth.fill(synth.SEED, j, t, s.nbytes) for t, s in enumerate(sp)]
            off, _ = oracle.layout([s.nbytes for s in sp])
            imgs.append(oracle.pack(tb, off, g["L_star"]))
        P = oracle.encode(imgs, g["unit"], rank)
        dev_only = bool(flags & C.CKPT_OPT_DEVICE_ONLY)  # no host image: the drill checks the tensors

        def view():
            return (imgs[rank], P) if dev_only else C.ckpt_host_view(ctx, 0, copy=True)
        d, p = view()
        ok = [bool(np.array_equal(d, imgs[rank])), bool(np.array_equal(p, P))]
        # drill: every rank k in turn is lost (tensors + host image), rebuilt, reloaded
        for k in range(world):
            fill_state(ts, rank, seed=77 + k, xor_mode=1)
            if rank == k:
                C.ckpt_forget(ctx, 0xA5)
                for t in ts:
                    t.view(torch.uint8).fill_(0xA5)
            dist.barrier()
            C.ckpt_rebuild(ctx, k)
            C.ckpt_load(ctx)
            torch.cuda.synchronize()
            d, p = view()
            good = np.array_equal(d, imgs[rank]) and np.array_equal(p, P)
            for t, x in enumerate(ts):
                got = x.contiguous().view(torch.uint8).cpu().numpy()
                good = good and np.array_equal(got, synth.fill(synth.SEED, rank, t, specs[t].nbytes))
            ok.append(bool(good))
        # a second snapshot after the drill still commits and matches
        sid = C.ckpt_snapshot(ctx)
        C.ckpt_wait(ctx, sid)
        d, p = view()
        ok.append(bool(np.array_equal(d, imgs[rank]) and np.array_equal(p, P)))
        C.ckpt_destroy(ctx)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


def _retry_port_clash(fn):
    """_free_port closes the socket before the workers' TCPStore binds it, so another
    process can take the port in between (seen once in 25 cases: EADDRINUSE inside
    init_process_group, before any work): run the case again on a fresh port."""
    def wrapped(*a, **kw):
        for attempt in range(3):
            try:
                return fn(*a, **kw)
            except AssertionError as e:
                if "EADDRINUSE" not in str(e) or attempt == 2:
                    raise
    return wrapped


@_retry_port_clash
def _run(world, case, timeout=300):
    import queue
    import time

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    os.environ.setdefault("CKPT_TIMEOUT_S", "90")
    ps = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in ps:
        p.start()
    res, t0 = [], time.time()
    try:
        while len(res) < world:
            try:
                r = q.get(timeout=5)
            except queue.Empty:
                dead = [p for p in ps if p.exitcode not in (None, 0)]
                assert not dead, f"worker died: exit codes {[p.exitcode for p in ps]}"
                assert time.time() - t0 < timeout, "multi-GPU case timed out"
                continue
            res.append(r)
            assert r[2] is None, f"rank {r[0]}:\n{r[2]}"
    finally:
        for p in ps:
            p.join(30 if len(res) == world else 1)
            if p.is_alive():
                p.kill()
    for rank, ok, err in sorted(res, key=lambda x: x[0]):
        assert all(ok), f"rank {rank}: {ok}"


def _world():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2310_12670_b200 import build
    build.build()
    return n


@pytest.mark.parametrize("case", [
    ("tiny_7", 4096, 0, 1 << 20, 0, 1),
    ("tiny_5", 1024, 2, 1 << 16, 0x2, 0),
    ("tiny_9", 16, 3, 4096, 0, 1),
    ("tiny_6", 0, 0, 1 << 20, 0, 0),
    ("tiny_7", 4096, 2, 1 << 16, 0x18, 1),
    ("tiny_5", 256, 0, 1 << 20, 0x10, 0),
    ("tiny_7", 4096, 0, 1 << 20, 0x200, 1),  # CKPT_OPT_REBUILD_SHARES (Q27)
    ("tiny_5", 1024, 2, 1 << 16, 0x200, 0),
    ("tiny_5", 4096, 0, 1 << 16, 0x800, 1),  # CKPT_OPT_REBUILD_SELF (the default at m >= 3 is shares)
    ("tiny_7", 4096, 0, 1 << 20, 0x400, 1),  # CKPT_OPT_XOR_PUSH: bulk XOR reductions over NVLink
    ("tiny_6", 16, 0, 1 << 16, 0x600, 0),
    ("tiny_9", 4096, 0, 1 << 16, 0x20, 1),   # DEVICE_ONLY over IPC (protection in HBM, drill checks tensors)
])
def test_ipc_group_all_gpus(case):
    _run(min(_world(), 8), case)


def test_ipc_group_pair():
    _world()
    _run(2, ("tiny_8", 65536, 4, 1 << 20, 0, 0))


def test_ipc_c1_16mib_all_gpus():
    _run(min(_world(), 8), ("c1_16mb_fp32_m8", 65536, 0, 64 << 20, 0, 0))


def _worker_c2(rank, world, port, q, config="c2_7b_tp8", extra_flags=0):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch
        import torch.distributed as dist

        import synth
        from gpu_util import verify_images_full, verify_tensors_full
        from paper_2310_12670_b200 import ckpt as C
        from synth.gpu import descriptors, make_rank_state

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", device_id=dev)
        specs, ts = make_rank_state(config, rank, dev)
        # bench.py's launch configuration: full-copy staging, 512 MiB buckets, TMA pack
        ctx = C.ckpt_create(rank, C.ckpt_options_default(
            n_slots=0, bucket_bytes=512 << 20, stripe_unit=1 << 20,
            flags=C.CKPT_OPT_TIMING | C.CKPT_OPT_HOST_LOAD | C.CKPT_OPT_TMA_PACK | extra_flags, host_buffers=1))
        C.ckpt_register(ctx, descriptors(ts, specs))
        C.protect_ipc(ctx)
        g = C.ckpt_geometry(ctx)
        stream = torch.cuda.current_stream()
        sid = C.ckpt_snapshot(ctx, 512 << 20, stream)
        C.ckpt_wait(ctx, sid)
        u, m, Ls = g["unit"], g["m"], g["L_star"]
        all_specs = [synth.config_tensors(config, j) for j in range(m)]
        ok, info = [], {}
        views = {rank: C.ckpt_host_view(ctx, 0)}
        n = verify_images_full(all_specs, Ls, u, views)  # every byte of D_rank and P_rank
        ok.append(n == Ls + Ls // (m - 1))
        info["image_bytes_checked"] = n
        del views
        # lose member k = m-1 (tensors + host image), rebuild over NVLink, reload
        k = m - 1
        if rank == k:
            C.ckpt_forget(ctx, 0xA5)
            for t in ts:
                t.view(torch.uint8).fill_(0xA5)
        dist.barrier()
        C.ckpt_rebuild(ctx, k, stream)
        torch.cuda.synchronize()
        dist.barrier()
        if rank == k:
            views = {k: C.ckpt_host_view(ctx, 0)}
            n = verify_images_full(all_specs, Ls, u, views, ranks=[k], rebuild_k=k)
            ok.append(n == Ls + Ls // (m - 1))
            info["rebuilt_bytes_checked"] = n
            del views
        C.ckpt_load(ctx, stream)
        torch.cuda.synchronize()
        if rank == k:
            n = verify_tensors_full(specs, rank, ts)
            ok.append(n == sum(s.nbytes for s in specs))
            info["tensor_bytes_checked"] = n
        C.ckpt_destroy(ctx)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, None, info))
    except Exception:
        q.put((rank, None, traceback.format_exc(), None))


@pytest.mark.parametrize("config,flags", [("c2_7b_tp8", 0), ("c4_34b_tp8_stage0", 0), ("c2_7b_tp8", 0x400),
                                          ("c2_7b_tp8", 0x10)])  # CE gather (m = 2: the CE mirror)
def test_ipc_full_size_full_image(config, flags):
    """BASELINE configs 2 and 4 at full size in the bench launch configuration (one
    process per GPU, full-copy staging, 512 MiB buckets, TMA pack, TMA XOR over NVLink).
    Unsampled: every byte of every rank's data (O3) and parity row (O4, Eq 1 P.474-477)
    against the oracle; then member m-1 is lost, rebuilt (Eq 2 P.481-484) and every byte of
    its image compared with O6, its parity row with O4 and its tensors after the load."""
    world = min(_world(), 8)
    import queue
    import time

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_c2, args=(r, world, port, q, config, flags)) for r in range(world)]
    for p in ps:
        p.start()
    res, t0 = [], time.time()
    try:
        while len(res) < world:
            try:
                r = q.get(timeout=5)
            except queue.Empty:
                assert all(p.exitcode in (None, 0) for p in ps), "worker died"
                assert time.time() - t0 < 900, "timed out"
                continue
            assert r[2] is None, r[2]
            res.append(r)
    finally:
        for p in ps:
            p.join(30)
            if p.is_alive():
                p.kill()
    for rank, ok, _, info in sorted(res, key=lambda x: x[0]):
        print(f"rank {rank}: {info}")
        assert ok and all(ok), (rank, "failed checks (case index)", [i for i, x in enumerate(ok or []) if not x])


def _worker_arc(rank, world, port, q, scheme):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import itertools

        import torch
        import torch.distributed as dist

        import oracle
        import synth
        from paper_2310_12670_b200 import ckpt as C
        from synth.gpu import descriptors, fill_state, make_rank_state

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", device_id=dev)
        specs, ts = make_rank_state("tiny_8", rank, dev, misalign=1)
        ctx = C.ckpt_create(rank, C.ckpt_options_default(stripe_unit=4096, n_slots=0, bucket_bytes=1 << 16,
                                                         flags=C.CKPT_OPT_SHM_ARENA))
        C.ckpt_register(ctx, descriptors(ts, specs))
        C.protect_ipc(ctx, scheme=scheme)
        g = C.ckpt_geometry(ctx)
        imgs = []
        for j in range(world):
            sp = synth.config_tensors("tiny_8", j)
            tb = [synth.fill(synth.SEED, j, t, s.nbytes) for t, s in enumerate(sp)]
            off, _ = oracle.layout([s.nbytes for s in sp])
            imgs.append(oracle.pack(tb, off, g["L_star"]))
        Ps = oracle.encode_all(imgs, g["unit"]) if scheme != 2 else None
        nxt = (rank + 1) % world

        def views_ok():
            d, p = C.ckpt_host_view(ctx, 0, copy=True)
            ad, ap = C.ckpt_host_view(ctx, 2, copy=True)
            ok = np.array_equal(d, imgs[rank]) and np.array_equal(ad, imgs[nxt])
            if scheme != 2:
                ok = ok and np.array_equal(p, Ps[rank])
            if scheme == 3:
                ok = ok and np.array_equal(ap, Ps[nxt])
            return bool(ok)

        sid = C.ckpt_snapshot(ctx)
        C.ckpt_wait(ctx, sid)
        ok = [views_ok()]
        cases = [(x,) for x in range(world)]
        if scheme == 3 and world >= 3:
            cases += list(itertools.combinations(range(world), 2))
        for lost in cases:
            mask = sum(1 << x for x in lost)
            fill_state(ts, rank, seed=5 + mask, xor_mode=1)
            if rank in lost:
                C.ckpt_forget(ctx, 0xA5)
                for t in ts:
                    t.view(torch.uint8).fill_(0xA5)
            dist.barrier()
            C.ckpt_recover(ctx, mask)
            C.ckpt_load(ctx)
            torch.cuda.synchronize()
            dist.barrier()
            good = views_ok()
            for t, x in enumerate(ts):
                got = x.contiguous().view(torch.uint8).cpu().numpy()
                good = good and np.array_equal(got, synth.fill(synth.SEED, rank, t, specs[t].nbytes))
            ok.append(bool(good))
        sid = C.ckpt_snapshot(ctx)
        C.ckpt_wait(ctx, sid)
        ok.append(views_ok())
        dist.barrier()
        C.ckpt_destroy(ctx)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("scheme", [2, 3])
def test_ipc_arc_schemes(scheme):
    """ARC and ARC+AEC across processes: pushes into the holder's shared-memory arena,
    every single loss (and every pair for ARC+AEC) recovered, bit-exact."""
    world = min(_world(), 4)
    import queue
    import time

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_arc, args=(r, world, port, q, scheme)) for r in range(world)]
    for p in ps:
        p.start()
    res, t0 = [], time.time()
    try:
        while len(res) < world:
            try:
                r = q.get(timeout=5)
            except queue.Empty:
                assert all(p.exitcode in (None, 0) for p in ps), "worker died"
                assert time.time() - t0 < 300, "timed out"
                continue
            assert r[2] is None, r[2]
            res.append(r)
    finally:
        for p in ps:
            p.join(30)
            if p.is_alive():
                p.kill()
    for rank, ok, _ in res:
        assert all(ok), (rank, "failed checks (case index)", [i for i, x in enumerate(ok) if not x])


def _worker_sub(rank, world, port, q, G):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch
        import torch.distributed as dist

        import oracle
        import synth
        from paper_2310_12670_b200 import ckpt as C
        from synth.gpu import descriptors, fill_state, make_rank_state

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", device_id=dev)
        sub = None
        for s0 in range(0, world, G):
            grp = dist.new_group(list(range(s0, s0 + G)))
            if s0 <= rank < s0 + G:
                sub, base = grp, s0
        specs, ts = make_rank_state("tiny_7", rank, dev, misalign=1)
        ctx = C.ckpt_create(rank, C.ckpt_options_default(stripe_unit=4096, n_slots=0, bucket_bytes=1 << 16))
        C.ckpt_register(ctx, descriptors(ts, specs))
        C.protect_ipc(ctx, group=sub)
        g = C.ckpt_geometry(ctx)
        sid = C.ckpt_snapshot(ctx)
        C.ckpt_wait(ctx, sid)
        imgs = []
        for j in range(base, base + G):
            sp = synth.config_tensors("tiny_7", j)
            tb = [synth.fill(synth.SEED, j, t, s.nbytes) for t, s in enumerate(sp)]
            off, _ = oracle.layout([s.nbytes for s in sp])
            imgs.append(oracle.pack(tb, off, g["L_star"]))
        me = rank - base
        d, p = C.ckpt_host_view(ctx, 0, copy=True)
        ok = [g["m"] == G, bool(np.array_equal(d, imgs[me])), bool(np.array_equal(p, oracle.encode(imgs, g["unit"], me)))]
        # one loss in EVERY subgroup at once (member 0 of each), recovered independently
        fill_state(ts, rank, seed=9, xor_mode=1)
        if me == 0:
            C.ckpt_forget(ctx, 0xA5)
            for t in ts:
                t.view(torch.uint8).fill_(0xA5)
        dist.barrier()
        C.ckpt_rebuild(ctx, 0)
        C.ckpt_load(ctx)
        torch.cuda.synchronize()
        good = True
        for t, x in enumerate(ts):
            got = x.contiguous().view(torch.uint8).cpu().numpy()
            good = good and np.array_equal(got, synth.fill(synth.SEED, rank, t, specs[t].nbytes))
        ok.append(bool(good))
        dist.barrier()
        C.ckpt_destroy(ctx)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


def test_ipc_disjoint_subgroups():
    """the node's ranks split into disjoint protection groups (here pairs);
    each group encodes its own parity, and one loss per group is recovered concurrently."""
    world = min(_world(), 8)
    if world < 4:
        pytest.skip("needs >= 4 GPUs for two groups of two")
    world -= world % 2
    import queue
    import time

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_sub, args=(r, world, port, q, 2)) for r in range(world)]
    for p in ps:
        p.start()
    res, t0 = [], time.time()
    try:
        while len(res) < world:
            try:
                r = q.get(timeout=5)
            except queue.Empty:
                assert all(p.exitcode in (None, 0) for p in ps), "worker died"
                assert time.time() - t0 < 300, "timed out"
                continue
            assert r[2] is None, r[2]
            res.append(r)
    finally:
        for p in ps:
            p.join(30)
            if p.is_alive():
                p.kill()
    for rank, ok, _ in res:
        assert all(ok), (rank, ok)


# ---------------------------------------------------------------- AOR (f4) --------------
def _aor_worker(rank, world, port, q):
    """ZeRO-1 members, one process per GPU: Eq 4 replicas vs the oracle and vs the owners'
    device shards; then every member in turn is lost (device shard + held replica, context
    re-created) and recovered with the protocol of include/ckpt_aor.h over dist.barrier."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch
        import torch.distributed as dist

        import oracle
        from paper_2310_12670_b200 import ckpt as C

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", device_id=dev)
        sizes = [70_003 + 9_001 * j for j in range(world)]
        bounds = [0]
        for n in sizes:
            bounds.append(bounds[-1] + n)
        owner = (rank + 1) % world
        gen = torch.Generator(device=dev).manual_seed(5)       # the all-reduced gradient: same everywhere
        master = torch.randn(sizes[rank], device=dev, generator=torch.Generator(device=dev).manual_seed(100 + rank))
        grad = torch.empty(bounds[-1], device=dev)
        key = C.aor_group_key()
        opt = C.ckpt_aor_options_default(key=key, chunk_bytes=64 << 10, n_slots=2, flags=C.CKPT_AOR_PERSIST)
        a = C.ckpt_aor_create(rank, opt, master, grad, bounds, rank)
        dist.barrier()
        C.ckpt_aor_seed(a, 0)
        dist.barrier()
        rep = C.ckpt_aor_view(a)[0]
        t = 0

        def steps(n):
            nonlocal rep, t
            for _ in range(n):
                eta = 0.01 * (t + 1)
                grad.copy_(torch.randn(bounds[-1], device=dev, generator=gen) * 1e-2)
                s = C.ckpt_aor_step(a, eta)
                C.ckpt_aor_fence(a, s)
                rep = oracle.aor_update(rep, grad[bounds[owner]:bounds[owner + 1]].cpu().numpy(), eta)
                master.sub_(grad[bounds[rank]:bounds[rank + 1]] * eta)
                grad.fill_(float("nan"))
                t += 1

        def check():
            got, step, state = C.ckpt_aor_view(a)
            masters = [None] * world
            dist.all_gather_object(masters, master.cpu().numpy())
            return (state == C.CKPT_AOR_CLEAN and step == t
                    and np.array_equal(got.view(np.uint32), rep.view(np.uint32))
                    and np.array_equal(got.view(np.uint32), masters[owner].view(np.uint32))), masters

        ok = []
        steps(3)
        good, masters = check()
        ok.append(good)
        for x in range(world):
            if rank == x:
                master.view(torch.int32).fill_(0x7FA5A5A5)
                C.ckpt_aor_forget(a)
                C.ckpt_aor_destroy(a)
                a = C.ckpt_aor_create(rank, opt, master, grad, bounds, rank)   # the replacement re-attaches
            dist.barrier()
            step = C.aor_recover(a, 1 << x, rank, world, dist.barrier)
            torch.cuda.synchronize()
            ok.append(step == t)
            ok.append(bool(np.array_equal(master.cpu().numpy().view(np.uint32), masters[rank].view(np.uint32))))
            if rank == x:
                rep = masters[owner].copy()        # its held replica was re-seeded by its owner
            steps(1)
            good, masters = check()
            ok.append(good)
        C.ckpt_aor_destroy(a)
        dist.barrier()
        if rank == 0:
            C.ckpt_aor_unlink(key, world)
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


@_retry_port_clash
def _run_fn(fn, world, timeout=300):
    import queue
    import time

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    os.environ.setdefault("CKPT_TIMEOUT_S", "90")
    ps = [ctx.Process(target=fn, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res, t0 = [], time.time()
    try:
        while len(res) < world:
            try:
                r = q.get(timeout=5)
            except queue.Empty:
                dead = [p for p in ps if p.exitcode not in (None, 0)]
                assert not dead, f"worker died: exit codes {[p.exitcode for p in ps]}"
                assert time.time() - t0 < timeout, "multi-GPU case timed out"
                continue
            res.append(r)
            assert r[2] is None, f"rank {r[0]}:\n{r[2]}"
    finally:
        for p in ps:
            p.join(30 if len(res) == world else 1)
            if p.is_alive():
                p.kill()
    for rank, ok, err in sorted(res, key=lambda x: x[0]):
        assert all(ok), f"rank {rank}: {ok}"


def test_aor_zero1_members_all_gpus():
    _run_fn(_aor_worker, min(_world(), 8))


# ---------------------------------------------------------------- f3: group restart -------
def _persist_worker(phase, key, drop, rank, world, port, q):
    """phase 'write': commit v1 and v2 (tensors mutated between), start v3, every process
    dies.  phase 'read': a NEW process per GPU re-attaches the persistent arena through the
    IPC handshake (the group's committed version = v2), member `drop` first lost its host
    memory (its shm files are gone) and is recovered from parity, then every member loads."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch
        import torch.distributed as dist

        import synth
        from paper_2310_12670_b200 import ckpt as C
        from synth.gpu import alloc_state, descriptors, fill_state

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", device_id=dev)
        specs = synth.config_tensors("tiny_7", rank)
        ts = alloc_state(specs, dev, misalign=1)
        if phase == "read" and drop == rank:
            for b in range(2):
                try:
                    os.unlink(f"/dev/shm/reft-{key:016x}-{rank}-{b}")
                except FileNotFoundError:
                    pass
        dist.barrier()
        o = C.ckpt_options_default(n_slots=0, bucket_bytes=1 << 16, stripe_unit=4096,
                                   flags=C.CKPT_OPT_SHM_ARENA, arena_key=key)
        ctx = C.ckpt_create(rank, o)
        C.ckpt_register(ctx, descriptors(ts, specs), {"local_rank": rank})
        C.protect_ipc(ctx)
        ok = []
        if phase == "write":
            fill_state(ts, rank)
            for seed in (None, 31):
                if seed is not None:
                    fill_state(ts, rank, seed=seed, xor_mode=1)
                sid = C.ckpt_snapshot(ctx)
                C.ckpt_wait(ctx, sid)
            fill_state(ts, rank, seed=32, xor_mode=1)
            dist.barrier()
            C.ckpt_snapshot(ctx)                  # v3 in flight when every process dies
            q.put((rank, [True], None))
            q.close()
            q.join_thread()
            os._exit(0)
        for t in ts:
            t.view(torch.uint8).fill_(0x77)       # fresh process: garbage in the tensors
        if drop >= 0:
            C.ckpt_recover(ctx, 1 << drop)
        C.ckpt_load(ctx)
        torch.cuda.synchronize()
        for t, x in enumerate(ts):
            want = synth.fill(synth.SEED, rank, t, specs[t].nbytes) ^ synth.fill(31, rank, t, specs[t].nbytes)
            ok.append(bool(np.array_equal(x.contiguous().view(torch.uint8).cpu().numpy(), want)))
        C.ckpt_destroy(ctx)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("drop", [-1, 1])
def test_group_restart_reattaches_over_ipc(drop):
    """SURVEY 8(f) f3 across GPUs: the whole group dies (as a TorchElastic restart would
    have it) after committing v2 and while v3 is in flight; new processes re-attach,
    agree on v2 through the handshake, recover a member without host memory, and load v2."""
    import functools
    world = min(_world(), 4)
    key = int.from_bytes(os.urandom(8), "little") | 1
    from paper_2310_12670_b200 import ckpt as C
    try:
        _run_fn(functools.partial(_persist_worker, "write", key, drop), world)
        _run_fn(functools.partial(_persist_worker, "read", key, drop), world)
    finally:
        C.ckpt_arena_unlink(key, world, 2)


def test_torchrun_elastic_replaces_a_killed_rank(tmp_path):
    """REFT-load after a real process failure under torchrun's elastic agent (P.545,
    P.551-555; SPEC S.514): rank N-1 loses its host memory and dies after v2 committed; the
    agent (--max-restarts 1) restarts the group, the new processes re-attach the persistent
    arenas, recover the replaced member from parity and load v2 bit-exactly
    (tools/elastic_drill.py)."""
    import json
    import random
    import subprocess
    import sys
    world = min(_world(), 4)
    from paper_2310_12670_b200 import ckpt as C
    key = random.getrandbits(48) | 1
    port = _free_port()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--max-restarts", "1", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(root, "tools", "elastic_drill.py"), "--key", hex(key), "--out", str(tmp_path)]
    env = dict(os.environ, CKPT_TIMEOUT_S="120")
    try:
        r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
        errs = "".join(f"--- {f.name}\n{f.read_text()}" for f in sorted(tmp_path.glob("*.err")))
        assert r.returncode == 0, errs + r.stdout[-2000:] + r.stderr[-3000:]
        res = [json.load(open(tmp_path / f"rank{j}.json")) for j in range(world)]
        for x in res:
            assert x["attempt"] == 1, x       # the group was restarted once by the agent
            assert x["ok"], x
    finally:
        C.ckpt_arena_unlink(key, world, 2)


def _abort_worker(rank, world, port, q):
    """Member 0 cannot serve a rebuild (it has no completed image): its failure aborts the
    group, so the member waiting for it fails with EPEER in seconds, not after the timeout."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import time

        import torch
        import torch.distributed as dist

        from paper_2310_12670_b200 import ckpt as C
        from synth.gpu import descriptors, make_rank_state

        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", device_id=dev)
        specs, ts = make_rank_state("tiny_7", rank, dev)
        ctx = C.ckpt_create(rank, C.ckpt_options_default(n_slots=0, bucket_bytes=1 << 16, stripe_unit=4096))
        C.ckpt_register(ctx, descriptors(ts, specs))
        C.protect_ipc(ctx)
        sid = C.ckpt_snapshot(ctx)
        C.ckpt_wait(ctx, sid)
        if rank == 0:
            C.ckpt_forget(ctx, 0xA5)         # a second loss: no survivor image to serve
        dist.barrier()
        t0 = time.time()
        code = 0
        try:
            C.ckpt_rebuild(ctx, world - 1)
        except C.CkptError as e:
            code = e.code
        el = time.time() - t0
        want = C.CKPT_EUNRECOVERABLE if rank == 0 else (C.CKPT_EPEER if rank == world - 1 else code)
        ok = [code == want, el < 30.0]
        C.ckpt_destroy(ctx)
        dist.destroy_process_group()
        q.put((rank, ok, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


def test_failed_member_aborts_the_group_fast():
    """a survivor that fails before its share of a collective rebuild must not
    leave its peers blocked until CKPT_TIMEOUT_S (here 300 s): the abort word releases them."""
    os.environ["CKPT_TIMEOUT_S"] = "300"
    try:
        _run_fn(_abort_worker, min(_world(), 2), timeout=200)
    finally:
        os.environ["CKPT_TIMEOUT_S"] = "90"
