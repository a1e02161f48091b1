"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, bit-exact.

Single-GPU cases use CKPT_GROUP_LOCAL groups (m contexts on cuda:0, the same kernels
and the same per-member stream schedule as the one-process-per-GPU IPC transport,
ordered with CUDA events instead of cross-process flags)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import assert_bytes_equal, need_gpu, oracle_image, oracle_tensor_bytes, tensor_bytes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    return need_gpu()


@pytest.fixture(scope="module")
def C(torch):
    from paper_2310_12670_b200 import ckpt
    return ckpt


def make_ctx(C, specs_ts, **opt):
    from synth.gpu import descriptors
    specs, ts = specs_ts
    o = C.ckpt_options_default(**opt)
    ctx = C.ckpt_create(0, o)
    C.ckpt_register(ctx, descriptors(ts, specs))
    return ctx


def tiny(rank, n=9, misalign=0, device="cuda:0"):
    from synth.gpu import alloc_state, fill_state
    specs = synth.config_tensors(f"tiny_{n}", rank)
    ts = alloc_state(specs, device, misalign)
    fill_state(ts, rank)
    return specs, ts


# ------------------------------------------------------------------ m = 1 ---------
@pytest.mark.parametrize("n_slots,bucket,flags", [
    (0, 0, 0), (2, 4096, 0), (4, 65536, 0), (3, 1 << 20, 0),
    (0, 0, 0x2), (2, 65536, 0x2), (4, 4096, 0x2),
    (0, 0, 0x8), (2, 65536, 0x8), (3, 4096, 0x8), (0, 0, 0x4), (0, 65536, 0x4)])
@pytest.mark.parametrize("misalign", [0, 1])
def test_snapshot_unprotected_matches_oracle(torch, C, n_slots, bucket, flags, misalign):
    st = tiny(0, n=11, misalign=misalign)
    specs, ts = st
    ctx = make_ctx(C, st, n_slots=n_slots, bucket_bytes=max(bucket, 4096), flags=flags)
    try:
        assert C.ckpt_protect(ctx, 1, 0) == C.CKPT_EUNAVAIL
        sid = C.ckpt_snapshot(ctx, bucket)
        C.ckpt_wait(ctx, sid)
        g = C.ckpt_geometry(ctx)
        want, off, L = oracle_image(specs, 0, g["L_star"])
        assert g["L"] == L == g["L_star"]
        data, par = C.ckpt_host_view(ctx, 0, copy=True)
        assert par is None
        assert_bytes_equal(data, want, "data image")
        assert [C.ckpt_tensor_offset(ctx, t) for t in range(len(specs))] == off
        # load: mutate the live tensors (a later step), restore, compare
        from synth.gpu import fill_state
        fill_state(ts, 0, seed=999, xor_mode=1)
        C.ckpt_load(ctx)
        torch.cuda.synchronize()
        for t, (x, w) in enumerate(zip(ts, oracle_tensor_bytes(specs, 0))):
            assert_bytes_equal(tensor_bytes(x), w, f"tensor {t} after load")
    finally:
        C.ckpt_destroy(ctx)


def test_register_errors(torch, C):
    ctx = C.ckpt_create(0)
    try:
        with pytest.raises(C.CkptError) as e:
            C.ckpt_register(ctx, [])
        assert e.value.code == C.CKPT_EINVAL
        x = torch.empty(0, device="cuda:0")
        with pytest.raises(C.CkptError):
            C.ckpt_register(ctx, [(x.data_ptr() or 16, 0, 0, 0, 0, "z")])
        h = torch.empty(16)  # host memory is rejected
        with pytest.raises(C.CkptError) as e:
            C.ckpt_register(ctx, [h])
        assert e.value.code == C.CKPT_EINVAL
        with pytest.raises(C.CkptError) as e:
            C.ckpt_load(ctx)
        assert e.value.code in (C.CKPT_ESTATE, C.CKPT_ENOSNAP)
    finally:
        C.ckpt_destroy(ctx)


def test_single_byte_tensor_and_busy(torch, C):
    x = torch.arange(1, dtype=torch.uint8, device="cuda:0") + 7
    ctx = C.ckpt_create(0, C.ckpt_options_default(n_slots=2, bucket_bytes=4096))
    try:
        C.ckpt_register(ctx, [x])
        sid = C.ckpt_snapshot(ctx)
        with pytest.raises(C.CkptError) as e:
            C.ckpt_snapshot(ctx)
        assert e.value.code == C.CKPT_EBUSY
        C.ckpt_wait(ctx, sid)
        d, _ = C.ckpt_host_view(ctx, 0, copy=True)
        assert d.size == 256 and d[0] == 7 and not d[1:].any()
    finally:
        C.ckpt_destroy(ctx)


# ------------------------------------------------------------------ LOCAL groups --
def make_group(torch, C, m, unit, n_slots=0, bucket=1 << 20, flags=0, misalign=0):
    states = [tiny(j, n=5 + j % 3, misalign=misalign) for j in range(m)]
    ctxs = [make_ctx(C, st, n_slots=n_slots, bucket_bytes=bucket, stripe_unit=unit, flags=flags)
            for st in states]
    C.protect_local(ctxs)
    return states, ctxs


@pytest.mark.parametrize("flag", [0x200, 0x800])
def test_rebuild_shares_flag_must_agree(torch, C, flag):
    """CKPT_OPT_REBUILD_SHARES / _SELF change who writes the lost member's parity row (Q27):
    a group whose members disagree would leave it unwritten or written twice -> EMISMATCH."""
    states = [tiny(j) for j in range(3)]
    ctxs = [make_ctx(C, st, n_slots=0, bucket_bytes=1 << 20, flags=flag if j == 1 else 0)
            for j, st in enumerate(states)]
    try:
        with pytest.raises(C.CkptError) as e:
            C.protect_local(ctxs)
        assert e.value.code == C.CKPT_EMISMATCH
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


@pytest.mark.parametrize("m,unit", [(2, 65536), (3, 4096), (4, 16), (8, 0)])
def test_push_encode_repeated_snapshots(torch, C, m, unit):
    """CKPT_OPT_XOR_PUSH: every row owner zeroes its parity before each snapshot and its
    peers XOR-reduce their units into it (Eq 1); three snapshots of changing state (the
    second would read P xor P = 0 if the zeroing were missing) each equal the oracle."""
    from synth.gpu import fill_state
    states, ctxs = make_group(torch, C, m, unit, 0, 1 << 16, flags=C.CKPT_OPT_XOR_PUSH, misalign=1)
    try:
        for step in range(3):
            if step:
                for j, (specs, ts) in enumerate(states):
                    fill_state(ts, j, seed=synth.SEED + step)  # a later training step
            snapshot_group(C, ctxs)
            g = C.ckpt_geometry(ctxs[0])
            Ds = [oracle_image(specs, j, g["L_star"], seed=synth.SEED + step)[0] for j, (specs, _) in enumerate(states)]
            Ps = oracle.encode_all(Ds, g["unit"])
            for j, c in enumerate(ctxs):
                d, p = C.ckpt_host_view(c, 0, copy=True)
                assert_bytes_equal(d, Ds[j], f"step {step} rank {j} data")
                assert_bytes_equal(p, Ps[j], f"step {step} rank {j} parity")
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


def test_xor_push_flag_must_agree(torch, C):
    """Push and pull encodes write a parity row differently (reductions from the peers vs a
    store by its owner): a group that mixes them is refused."""
    states = [tiny(j) for j in range(3)]
    ctxs = [make_ctx(C, st, n_slots=0, bucket_bytes=1 << 20, flags=C.CKPT_OPT_XOR_PUSH if j == 2 else 0)
            for j, st in enumerate(states)]
    try:
        with pytest.raises(C.CkptError) as e:
            C.protect_local(ctxs)
        assert e.value.code == C.CKPT_EMISMATCH
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


def snapshot_group(C, ctxs, bucket=0):
    ids = [C.ckpt_snapshot(c, bucket) for c in ctxs]
    for c, i in zip(ctxs, ids):
        C.ckpt_wait(c, i)


def expected_group(states, Lstar, unit):
    Ds = [oracle_image(specs, j, Lstar)[0] for j, (specs, _) in enumerate(states)]
    Ps = oracle.encode_all(Ds, unit) if len(Ds) > 1 else [None]
    return Ds, Ps


@pytest.mark.parametrize("m", [2, 3, 4, 8])
@pytest.mark.parametrize("unit,n_slots,bucket", [(65536, 0, 1 << 20), (4096, 3, 1 << 20), (16, 2, 4096),
                                                 (0, 0, 1 << 20), (65536, 4, 1 << 20)])
@pytest.mark.parametrize("flags", [0, 0x4, 0x10, 0x18, 0x400])
def test_group_encode_matches_oracle(torch, C, m, unit, n_slots, bucket, flags):
    if unit == 65536 and n_slots and (m - 1) * unit > bucket:
        pytest.skip("stripe larger than ring slot")
    states, ctxs = make_group(torch, C, m, unit, n_slots, bucket, flags=flags)
    try:
        snapshot_group(C, ctxs)
        g = C.ckpt_geometry(ctxs[0])
        Ls, ue = oracle.common_length([oracle.layout([s.nbytes for s in sp])[1] for sp, _ in states], unit)
        assert (g["L_star"], g["unit"], g["m"]) == (Ls, ue, m)
        Ds, Ps = expected_group(states, Ls, ue)
        for j, c in enumerate(ctxs):
            d, p = C.ckpt_host_view(c, 0, copy=True)
            assert_bytes_equal(d, Ds[j], f"rank {j} data")
            assert_bytes_equal(p, Ps[j], f"rank {j} parity")
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


@pytest.mark.parametrize("m,unit,n_slots,flags", [(2, 4096, 0, 0), (3, 4096, 2, 0), (4, 65536, 0, 0x2),
                                                  (8, 1024, 3, 0), (8, 0, 0, 0), (5, 64, 2, 0x2),
                                                  (4, 4096, 2, 0x18), (6, 256, 0, 0x18),
                                                  (4, 65536, 0, 0x80), (3, 4096, 0, 0x82), (5, 4096, 0, 0x88),
                                                  # CKPT_OPT_REBUILD_SHARES (Q27): survivors encode the lost row
                                                  (2, 4096, 0, 0x200), (4, 4096, 2, 0x200), (5, 65536, 0, 0x202),
                                                  (8, 1024, 3, 0x200), (3, 4096, 0, 0x280), (7, 16, 0, 0x200),
                                                  # CKPT_OPT_XOR_PUSH: push-mode encode (bulk XOR reductions)
                                                  (2, 4096, 0, 0x400), (4, 65536, 0, 0x402), (8, 1024, 0, 0x600),
                                                  (5, 16, 0, 0x480),
                                                  # CKPT_OPT_CE_GATHER at m = 2: the copy-engine mirror
                                                  (2, 4096, 0, 0x10), (2, 65536, 3, 0x10),
                                                  # CKPT_OPT_REBUILD_SELF at m >= 3 (the default there is shares)
                                                  (4, 4096, 2, 0x800), (5, 65536, 0, 0x802), (3, 4096, 0, 0x880),
                                                  (8, 1024, 0, 0x800)])
def test_group_drill_rebuild_every_rank(torch, C, m, unit, n_slots, flags):
    """Failure drill (Q12): rank k loses tensors and host image; rebuild + load."""
    from synth.gpu import fill_state
    states, ctxs = make_group(torch, C, m, unit, n_slots, bucket=max(1 << 16, (m - 1) * unit * 2), flags=flags,
                              misalign=1)
    try:
        snapshot_group(C, ctxs)
        g = C.ckpt_geometry(ctxs[0])
        Ds, Ps = expected_group(states, g["L_star"], g["unit"])
        for k in range(m):
            # later training steps mutate every rank; rank k is lost entirely
            for j, (specs, ts) in enumerate(states):
                fill_state(ts, j, seed=4242 + k, xor_mode=1)
            C.ckpt_forget(ctxs[k], 0xA5)
            for t in states[k][1]:
                t.view(torch.uint8).fill_(0xA5)
            with pytest.raises(C.CkptError) as e:
                C.ckpt_load(ctxs[k])
            assert e.value.code == C.CKPT_ENOSNAP
            for c in ctxs:
                C.ckpt_rebuild(c, k)
            d, p = C.ckpt_host_view(ctxs[k], 0, copy=True)
            assert_bytes_equal(d, Ds[k], f"rebuilt data of rank {k}")
            assert_bytes_equal(p, Ps[k], f"re-encoded parity of rank {k}")
            for c in ctxs:
                C.ckpt_load(c)
            torch.cuda.synchronize()
            for j, (specs, ts) in enumerate(states):
                for t, (x, w) in enumerate(zip(ts, oracle_tensor_bytes(specs, j))):
                    assert_bytes_equal(tensor_bytes(x), w, f"k={k}: rank {j} tensor {t} after load")
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


def test_two_losses_unrecoverable(torch, C):
    states, ctxs = make_group(torch, C, 4, 4096)
    try:
        snapshot_group(C, ctxs)
        C.ckpt_forget(ctxs[1])
        with pytest.raises(C.CkptError) as e:  # survivor 1 lost its image too
            C.ckpt_rebuild(ctxs[1], 0)
        assert e.value.code == C.CKPT_EUNRECOVERABLE
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


def test_bucket_size_invariance_and_commit(torch, C):
    """I8: images do not depend on the bucket size; commit keeps the previous image
    readable until the next snapshot is waited (P.553-554, S.431)."""
    from synth.gpu import fill_state
    # full-copy staging rounds buckets to lcm(stripe, 64 KiB) = 192 KiB here
    states, ctxs = make_group(torch, C, 4, 4096, n_slots=0)
    try:
        snapshot_group(C, ctxs, bucket=3 * 65536)
        first = [tuple(x.copy() for x in C.ckpt_host_view(c, 0, copy=True)) for c in ctxs]
        snapshot_group(C, ctxs, bucket=3 * 65536 * 3)
        for c, (d0, p0) in zip(ctxs, first):
            d, p = C.ckpt_host_view(c, 0, copy=True)
            assert_bytes_equal(d, d0, "data vs bucket size")
            assert_bytes_equal(p, p0, "parity vs bucket size")
        # mutate, snapshot, do NOT wait yet: completed still holds the old image
        for j, (_, ts) in enumerate(states):
            fill_state(ts, j, seed=7, xor_mode=1)
        ids = [C.ckpt_snapshot(c) for c in ctxs]
        for c, (d0, _) in zip(ctxs, first):
            assert_bytes_equal(C.ckpt_host_view(c, 0, copy=True)[0], d0, "completed image during snapshot")
        for c, i in zip(ctxs, ids):
            C.ckpt_wait(c, i)
        assert not np.array_equal(C.ckpt_host_view(ctxs[0], 0, copy=True)[0], first[0][0])
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


# ------------------------------------------------------------------ full sizes ----
def test_c1_16mib_m8_full_parity(torch, C):
    """BASELINE config 1: 8 ranks x 16 MiB fp32, encode + rebuild of every rank,
    compared element by element with the oracle (launch configuration of bench)."""
    from synth.gpu import make_rank_state, descriptors
    m = 8
    states = [make_rank_state("c1_16mb_fp32_m8", j, "cuda:0") for j in range(m)]
    ctxs = []
    for specs, ts in states:
        c = C.ckpt_create(0, C.ckpt_options_default(n_slots=0, stripe_unit=65536))  # a 16 MiB shard: small u
        C.ckpt_register(c, descriptors(ts, specs))
        ctxs.append(c)
    try:
        C.protect_local(ctxs)
        snapshot_group(C, ctxs)
        g = C.ckpt_geometry(ctxs[0])
        assert g["L_star"] == 16973824 and g["unit"] == 65536
        Ds, Ps = expected_group(states, g["L_star"], g["unit"])
        for j, c in enumerate(ctxs):
            d, p = C.ckpt_host_view(c, 0, copy=True)
            assert p.size == 2424832
            assert_bytes_equal(d, Ds[j], f"rank {j} data")
            assert_bytes_equal(p, Ps[j], f"rank {j} parity")
        for k in (0, 5, 7):
            C.ckpt_forget(ctxs[k])
            for c in ctxs:
                C.ckpt_rebuild(c, k)
            d, p = C.ckpt_host_view(ctxs[k], 0, copy=True)
            assert_bytes_equal(d, Ds[k], f"rebuilt rank {k}")
            assert_bytes_equal(p, Ps[k], f"re-encoded parity rank {k}")
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


BENCH_BUCKET = 512 << 20  # bench.py defaults: full-copy staging, 512 MiB buckets, TMA pack, u = 1 MiB


def bench_options(C, **kw):
    """The options bench.py's N=1 step runs with (bench.py main(): n_slots=0, 512 MiB
    buckets, CKPT_OPT_TMA_PACK -> pack_all_tma_kernel, CKPT_OPT_HOST_LOAD for e2e's load)."""
    o = dict(n_slots=0, bucket_bytes=BENCH_BUCKET, stripe_unit=1 << 20,
             flags=C.CKPT_OPT_TIMING | C.CKPT_OPT_HOST_LOAD | C.CKPT_OPT_TMA_PACK)
    o.update(kw)
    return C.ckpt_options_default(**o)


def test_c2_bench_config_full_image(torch, C):
    """BASELINE config 2 at full size in EXACTLY the configuration bench.py times at N=1
    (full-copy staging, 512 MiB buckets, the single-launch pack_all_tma_kernel, two host
    buffers): 1164 tensors, 11.8 GB.  Unsampled: every byte of the committed host image
    (both buffers, after the bench's warm-up pattern of repeated snapshots) against the
    oracle's O3 (P.369-371), then every byte of every tensor after ckpt_load from the host
    image (O7, P.545 step 1)."""
    from gpu_util import verify_images_full, verify_tensors_full
    from synth.gpu import make_rank_state, descriptors
    specs, ts = make_rank_state("c2_7b_tp8", 3, "cuda:0")
    assert len(specs) == 1164 and sum(s.nbytes for s in specs) == 11795488768
    ctx = C.ckpt_create(0, bench_options(C, host_buffers=2))
    try:
        C.ckpt_register(ctx, descriptors(ts, specs))
        assert C.ckpt_protect(ctx, 1, 0) == C.CKPT_EUNAVAIL
        stream = torch.cuda.current_stream()
        Ls = C.ckpt_geometry(ctx)["L_star"]
        for i in range(3):
            sid = C.ckpt_snapshot(ctx, BENCH_BUCKET, stream)
            C.ckpt_wait(ctx, sid)
            if i == 0:
                continue
            st = C.ckpt_get_stats(ctx)
            assert st["pack_launches"] == i + 1, "one pack launch per snapshot (single-launch TMA pack)"
            d, _ = C.ckpt_host_view(ctx, 0)  # the buffer just committed (i = 1, 2: both buffers)
            n = verify_images_full([specs], Ls, 1 << 20, {0: (d, None)}, gen_ranks=[3])
            assert n == Ls
            del d
        for t in ts:
            t.view(torch.uint8).fill_(0xA5)
        C.ckpt_load(ctx, stream)
        torch.cuda.synchronize()
        assert verify_tensors_full(specs, 3, ts) == sum(s.nbytes for s in specs)
    finally:
        C.ckpt_destroy(ctx)


@pytest.mark.parametrize("m,k,push", [(2, 1, 0), (3, 0, 0), (4, 2, 0), (4, 1, 1)])
def test_c2_group_full_image_and_rebuild(torch, C, m, k, push):
    """BASELINE config 2 at full size as an m-member protection group on one device
    (CKPT_GROUP_LOCAL: the same pack_all_tma_kernel and xor_tma_kernel<m-1> launches as the
    one-process-per-GPU product, full-copy staging, 512 MiB buckets, one host buffer).
    Unsampled: every byte of every member's data (O3) and parity row (O4, Eq 1 P.474-477)
    against the oracle; then member k is lost (tensors and host image poisoned), rebuilt
    (Eq 2 P.481-484) and every byte of its image compared with O6 and its parity row with
    O4; finally every byte of its tensors after ckpt_load (P.545)."""
    from gpu_util import verify_images_full, verify_tensors_full
    from synth.gpu import make_rank_state, descriptors
    free, _ = torch.cuda.mem_get_info()
    need = m * (2 * 11795488768 + 11795890176 // (m - 1)) + (4 << 30)
    if free < need:
        pytest.skip(f"needs {need / 1e9:.0f} GB of HBM, {free / 1e9:.0f} free")
    states, ctxs = [], []
    try:
        for j in range(m):
            specs, ts = make_rank_state("c2_7b_tp8", j, "cuda:0")
            states.append((specs, ts))
            o = bench_options(C, host_buffers=1)
            o.flags |= C.CKPT_OPT_XOR_PUSH if push else 0
            ctx = C.ckpt_create(0, o)
            ctxs.append(ctx)
            C.ckpt_register(ctx, descriptors(ts, specs))
        C.protect_local(ctxs)
        stream = torch.cuda.current_stream()
        ids = [C.ckpt_snapshot(c, BENCH_BUCKET, stream) for c in ctxs]
        for c, i in zip(ctxs, ids):
            C.ckpt_wait(c, i)
        g = C.ckpt_geometry(ctxs[0])
        Ls, u = g["L_star"], g["unit"]
        all_specs = [sp for sp, _ in states]
        views = {j: C.ckpt_host_view(ctxs[j], 0) for j in range(m)}
        n = verify_images_full(all_specs, Ls, u, views)
        assert n == m * (Ls + Ls // (m - 1))
        del views
        specs_k, ts_k = states[k]
        C.ckpt_forget(ctxs[k], 0xA5)
        for t in ts_k:
            t.view(torch.uint8).fill_(0xA5)
        for c in ctxs:
            C.ckpt_rebuild(c, k, stream)
        torch.cuda.synchronize()
        views = {j: C.ckpt_host_view(ctxs[j], 0) for j in range(m)}
        n = verify_images_full(all_specs, Ls, u, views, ranks=[k], rebuild_k=k)
        assert n == Ls + Ls // (m - 1)
        del views
        C.ckpt_load(ctxs[k], stream)
        torch.cuda.synchronize()
        assert verify_tensors_full(specs_k, k, ts_k) == sum(s.nbytes for s in specs_k)
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


@pytest.mark.parametrize("m,unit,flags", [(1, 65536, 0x20), (3, 4096, 0x20), (4, 65536, 0x22), (8, 1024, 0x28),
                                          (5, 256, 0x30), (4, 4096, 0x220), (6, 256, 0x230)])
def test_device_only_drill(torch, C, m, unit, flags):
    """DEVICE_ONLY: the image and parity stay in HBM; every lost rank is rebuilt from
    the survivors' device images and reloaded bit-exactly."""
    from synth.gpu import fill_state
    states = [tiny(j, n=6 + j % 2, misalign=1) for j in range(m)]
    ctxs = [make_ctx(C, st, n_slots=0, bucket_bytes=1 << 16, stripe_unit=unit, flags=flags) for st in states]
    try:
        if m == 1:
            assert C.ckpt_protect(ctxs[0], 1, 0) == C.CKPT_EUNAVAIL
        else:
            C.protect_local(ctxs)
        snapshot_group(C, ctxs)
        with pytest.raises(C.CkptError):
            C.ckpt_host_view(ctxs[0], 0)
        for k in range(m):
            for j, (_, ts) in enumerate(states):
                fill_state(ts, j, seed=31 + k, xor_mode=1)
            if m > 1:
                C.ckpt_forget(ctxs[k], 0x5A)
                for t in states[k][1]:
                    t.view(torch.uint8).fill_(0x5A)
                for c in ctxs:
                    C.ckpt_rebuild(c, k)
            for c in ctxs:
                C.ckpt_load(c)
            torch.cuda.synchronize()
            for j, (specs, ts) in enumerate(states):
                for t, (x, w) in enumerate(zip(ts, oracle_tensor_bytes(specs, j))):
                    assert_bytes_equal(tensor_bytes(x), w, f"k={k}: rank {j} tensor {t}")
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


def test_ring_bucket_sizes_match_full_copy(torch, C):
    """I8 across staging modes: ring slots with 4 different bucket sizes give the same
    images as the full-copy single-launch pack."""
    ref = None
    for n_slots, bucket in [(0, 1 << 20), (2, 12288), (3, 12288 * 5), (2, 12288 * 40)]:
        states, ctxs = make_group(torch, C, 4, 4096, n_slots=n_slots, bucket=max(bucket, 4096))
        try:
            snapshot_group(C, ctxs, bucket=bucket)
            imgs = [C.ckpt_host_view(c, 0, copy=True) for c in ctxs]
        finally:
            for c in ctxs:
                C.ckpt_destroy(c)
        if ref is None:
            ref = imgs
        for j, ((d, p), (d0, p0)) in enumerate(zip(imgs, ref)):
            assert_bytes_equal(d, d0, f"rank {j} data, slots={n_slots} bucket={bucket}")
            assert_bytes_equal(p, p0, f"rank {j} parity, slots={n_slots} bucket={bucket}")


@pytest.mark.parametrize("n_slots,m", [(0, 1), (2, 1), (0, 3), (3, 3)])
def test_fence_and_capture_point(torch, C, n_slots, m):
    """Q10: the snapshot holds the tensors as of the caller stream's position at
    ckpt_snapshot; after ckpt_fence the caller may mutate them on that stream while the
    D2H is still running, and the committed image is unaffected."""
    from synth.gpu import fill_state
    states = [tiny(j, n=7) for j in range(m)]
    ctxs = [make_ctx(C, st, n_slots=n_slots, bucket_bytes=12288 if n_slots else 1 << 20, stripe_unit=4096)
            for st in states]
    s = torch.cuda.Stream()
    try:
        if m == 1:
            C.ckpt_protect(ctxs[0], 1, 0)
        else:
            C.protect_local(ctxs)
        with torch.cuda.stream(s):
            # enqueued BEFORE the snapshot on the same stream: must be captured
            for j, (_, ts) in enumerate(states):
                fill_state(ts, j, seed=5, xor_mode=1, stream=s)
            ids = [C.ckpt_snapshot(c, 0, s) for c in ctxs]
            for c, i in zip(ctxs, ids):
                C.ckpt_fence(c, i, s)
            # enqueued AFTER the fence: must NOT be captured
            for j, (_, ts) in enumerate(states):
                fill_state(ts, j, seed=6, xor_mode=1, stream=s)
        for c, i in zip(ctxs, ids):
            C.ckpt_wait(c, i)
        for j, ((specs, _), c) in enumerate(zip(states, ctxs)):
            want = []
            for t, sp in enumerate(specs):
                w = oracle.fill(synth.SEED, j, t, sp.nbytes) ^ oracle.fill(5, j, t, sp.nbytes)
                want.append(w)
            off, L = oracle.layout([sp.nbytes for sp in specs])
            d, _ = C.ckpt_host_view(c, 0, copy=True)
            assert_bytes_equal(d[:L], oracle.pack(want, off, L), f"rank {j} image at the capture point")
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


@pytest.mark.parametrize("flags", [0, 0x2, 0x4, 0x8])
@pytest.mark.parametrize("n_slots", [0, 2])
def test_no_writes_outside_tensors(torch, C, flags, n_slots):
    """Bounds check without compute-sanitizer (closed on this pool): every tensor is a
    view with 64..79 canary bytes on both sides inside its own allocation; snapshot,
    rebuild and load (unpack) must leave every canary intact, for odd sizes and every
    misalignment mod 16."""
    from synth.gpu import descriptors, fill_state
    m = 3
    canary = 0x3C
    states, bases = [], []
    rng = np.random.default_rng(7)
    for j in range(m):
        specs = synth.config_tensors("tiny_9", j)
        ts, bs = [], []
        for i, s in enumerate(specs):
            pre = 64 + (i * 3 + j) % 16
            b = torch.full((pre + s.nbytes + 79,), canary, dtype=torch.uint8, device="cuda:0")
            bs.append((b, pre))
            ts.append(b[pre:pre + s.nbytes])
        fill_state(ts, j)
        states.append((specs, ts))
        bases.append(bs)
    ctxs = []
    for specs, ts in states:
        c = C.ckpt_create(0, C.ckpt_options_default(n_slots=n_slots, bucket_bytes=12288 if n_slots else 1 << 20,
                                                    stripe_unit=4096, flags=flags))
        C.ckpt_register(c, [C.tensor_desc(t, name=s.name) for t, s in zip(ts, specs)])
        ctxs.append(c)
    try:
        C.protect_local(ctxs)
        snapshot_group(C, ctxs)
        C.ckpt_forget(ctxs[1])
        for c in ctxs:
            C.ckpt_rebuild(c, 1)
        for j, (_, ts) in enumerate(states):
            fill_state(ts, j, seed=3, xor_mode=1)
        for c in ctxs:
            C.ckpt_load(c)
        torch.cuda.synchronize()
        for j, (specs, ts) in enumerate(states):
            for i, ((b, pre), s) in enumerate(zip(bases[j], specs)):
                h = b.cpu().numpy()
                assert (h[:pre] == canary).all() and (h[pre + s.nbytes:] == canary).all(), f"rank {j} tensor {i}"
                assert_bytes_equal(h[pre:pre + s.nbytes], oracle.fill(synth.SEED, j, i, s.nbytes), f"rank {j} tensor {i}")
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


def _arc_expect(states, Lstar, unit, scheme):
    Ds = [oracle_image(specs, j, Lstar)[0] for j, (specs, _) in enumerate(states)]
    Ps = oracle.encode_all(Ds, unit) if scheme != 2 else [None] * len(Ds)
    MDs = [oracle.arc_copy(Ds, i) for i in range(len(Ds))]
    MPs = [Ps[(i + 1) % len(Ds)] for i in range(len(Ds))]
    return Ds, Ps, MDs, MPs


def _check_all_views(C, ctxs, exp, scheme, what):
    Ds, Ps, MDs, MPs = exp
    for j, c in enumerate(ctxs):
        d, p = C.ckpt_host_view(c, 0, copy=True)
        assert_bytes_equal(d, Ds[j], f"{what}: member {j} data")
        if scheme != 2:
            assert_bytes_equal(p, Ps[j], f"{what}: member {j} parity")
        ad, ap = C.ckpt_host_view(c, 2, copy=True)
        assert_bytes_equal(ad, MDs[j], f"{what}: member {j} ARC copy of {(j + 1) % len(ctxs)}")
        if scheme == 3:
            assert_bytes_equal(ap, MPs[j], f"{what}: member {j} ARC parity copy")


@pytest.mark.parametrize("m,scheme", [(2, 2), (3, 2), (4, 2), (3, 3), (4, 3), (5, 3), (8, 3)])
def test_arc_schemes_snapshot_and_every_recovery(torch, C, m, scheme):
    """ARC (ring copies, 2 W_n/m) and ARC+AEC (collaborative, any two
    losses for m >= 3) -- host images, parity rows and ARC copies bit-exact against the
    oracle; every single loss and (ARC+AEC) every pair recovered and reloaded."""
    import itertools

    from synth.gpu import fill_state
    unit = 4096
    states = [tiny(j, n=5 + j % 3, misalign=1) for j in range(m)]
    ctxs = [make_ctx(C, st, n_slots=0, bucket_bytes=1 << 16, stripe_unit=unit, flags=0x40) for st in states]
    try:
        C.protect_local(ctxs, scheme=scheme)
        snapshot_group(C, ctxs)
        g = C.ckpt_geometry(ctxs[0])
        exp = _arc_expect(states, g["L_star"], g["unit"], scheme)
        _check_all_views(C, ctxs, exp, scheme, "snapshot")
        cases = [(x,) for x in range(m)]
        if scheme == 3:
            cases += list(itertools.combinations(range(m), 2))
        for lost in cases:
            mask = sum(1 << x for x in lost)
            for j, (_, ts) in enumerate(states):
                fill_state(ts, j, seed=11 + mask, xor_mode=1)
            for x in lost:
                C.ckpt_forget(ctxs[x], 0xA5)
                for t in states[x][1]:
                    t.view(torch.uint8).fill_(0xA5)
            for c in ctxs:
                C.ckpt_recover(c, mask)
            _check_all_views(C, ctxs, exp, scheme, f"after losing {lost}")
            for c in ctxs:
                C.ckpt_load(c)
            torch.cuda.synchronize()
            for j, (specs, ts) in enumerate(states):
                for t, (x, w) in enumerate(zip(ts, oracle_tensor_bytes(specs, j))):
                    assert_bytes_equal(tensor_bytes(x), w, f"lost {lost}: member {j} tensor {t}")
        # a snapshot after the drills still commits the same images everywhere
        snapshot_group(C, ctxs)
        _check_all_views(C, ctxs, exp, scheme, "snapshot after drills")
        if m >= 3:  # beyond the scheme: consistent refusal, nothing changes
            bad = 0b11 if scheme == 2 else 0b111
            for c in ctxs:
                with pytest.raises(C.CkptError) as e:
                    C.ckpt_recover(c, bad)
                assert e.value.code == C.CKPT_EUNRECOVERABLE
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


def test_shm_arena_aec_matches_anon(torch, C):
    """The shared-memory arena (CKPT_OPT_SHM_ARENA) holds the same images as the
    anonymous one for the default AEC scheme."""
    states, ctxs = make_group(torch, C, 4, 4096, flags=0x40)
    try:
        snapshot_group(C, ctxs)
        g = C.ckpt_geometry(ctxs[0])
        Ds, Ps = expected_group(states, g["L_star"], g["unit"])
        for j, c in enumerate(ctxs):
            d, p = C.ckpt_host_view(c, 0, copy=True)
            assert_bytes_equal(d, Ds[j], f"rank {j} data")
            assert_bytes_equal(p, Ps[j], f"rank {j} parity")
    finally:
        for c in ctxs:
            C.ckpt_destroy(c)


def test_load_from_device_copy_and_host_path_agree(torch, C):
    """With full-copy staging, ckpt_load right after a commit restores from the device copy
    (no H2D); CKPT_OPT_HOST_LOAD restores from host memory -- same bytes, and the stats
    show which path ran."""
    from synth.gpu import fill_state
    for flags, expect_h2d in ((0, False), (0x80, True)):
        st = tiny(0, n=9, misalign=1)
        specs, ts = st
        ctx = make_ctx(C, st, n_slots=0, bucket_bytes=1 << 16, flags=flags)
        try:
            C.ckpt_protect(ctx, 1, 0)
            sid = C.ckpt_snapshot(ctx)
            C.ckpt_wait(ctx, sid)
            fill_state(ts, 0, seed=77, xor_mode=1)
            C.ckpt_stats_reset(ctx)
            C.ckpt_load(ctx)
            torch.cuda.synchronize()
            assert (C.ckpt_get_stats(ctx)["h2d_bytes"] > 0) == expect_h2d
            for t, (x, w) in enumerate(zip(ts, oracle_tensor_bytes(specs, 0))):
                assert_bytes_equal(tensor_bytes(x), w, f"flags={flags:#x} tensor {t}")
            # a snapshot in flight invalidates the device copy: load must refuse
            sid = C.ckpt_snapshot(ctx)
            with pytest.raises(C.CkptError):
                C.ckpt_load(ctx)
            C.ckpt_wait(ctx, sid)
        finally:
            C.ckpt_destroy(ctx)


def test_has_window_gates_the_d2h(torch, C):
    """HAS placement (Alg 1 layers): with CKPT_OPT_WINDOWED no bucket reaches host memory
    while the training stream holds the window closed; once reopened the snapshot
    completes and matches the oracle."""
    import time
    st = tiny(0, n=9)
    specs, ts = st
    ctx = make_ctx(C, st, n_slots=0, bucket_bytes=1 << 16, flags=C.CKPT_OPT_WINDOWED)
    s = torch.cuda.Stream()
    try:
        C.ckpt_protect(ctx, 1, 0)
        C.ckpt_window(ctx, False, s)
        sid = C.ckpt_snapshot(ctx, 0, s)
        time.sleep(0.3)
        d_ongoing, _ = C.ckpt_host_view(ctx, 1, copy=True)
        assert not d_ongoing.any(), "D2H ran while the window was closed"
        C.ckpt_window(ctx, True, s)
        C.ckpt_wait(ctx, sid)
        g = C.ckpt_geometry(ctx)
        want, _, _ = oracle_image(specs, 0, g["L_star"])
        assert_bytes_equal(C.ckpt_host_view(ctx, 0, copy=True)[0], want, "image after the window opened")
    finally:
        C.ckpt_destroy(ctx)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("n_slots", [0, 3])
def test_has_windowed_snapshot_of_many_buckets_never_blocks_the_caller(torch, C, n_slots):
    """HAS windows with thousands of buckets (256 MiB in 64 KiB buckets): ckpt_snapshot is
    issued while every window is closed and must return at once -- the training thread opens
    the windows only afterwards, so enqueueing every gated copy up front would fill a stream
    queue and block it forever (the 1F1B run's C3 hang).  The caller then runs a "training
    loop" of short open/closed window phases (ckpt_window tops up the gated copies) until
    ckpt_test reports completion; the committed image matches the oracle."""
    import time

    import synth
    from synth.gpu import alloc_state, fill_state
    specs = [synth.TensorSpec(f"t{i}", "fp32" if i % 2 else "bf16", (16 << 20) // (4 if i % 2 else 2) - 3 * i, "param")
             for i in range(16)]
    ts = alloc_state(specs, "cuda:0", 1)
    fill_state(ts, 0)
    ctx = make_ctx(C, (specs, ts), n_slots=n_slots, bucket_bytes=1 << 16, flags=C.CKPT_OPT_WINDOWED)
    s = torch.cuda.Stream()
    try:
        C.ckpt_protect(ctx, 1, 0)
        g = C.ckpt_geometry(ctx)
        assert g["L"] // (1 << 16) >= 4000
        C.ckpt_window(ctx, 0, s)
        t0 = time.perf_counter()
        sid = C.ckpt_snapshot(ctx, 0, s)
        assert time.perf_counter() - t0 < 20, "ckpt_snapshot blocked while the windows were closed"
        if n_slots:  # ring: later packs wait for earlier buckets' D2H, so the fence cannot be placed yet
            with pytest.raises(C.CkptError) as e:
                C.ckpt_fence(ctx, sid, s)
            assert e.value.code == C.CKPT_EBUSY
        else:        # full copy: every pack is already enqueued
            C.ckpt_fence(ctx, sid, s)
        phases, t1 = 0, time.perf_counter()
        while True:
            C.ckpt_window(ctx, C.CKPT_WINDOW_BUBBLE | C.CKPT_WINDOW_COMPUTE, s)
            torch.cuda._sleep(2_000_000)          # ~1 ms of "computation" with the window open
            C.ckpt_window(ctx, 0, s)
            torch.cuda._sleep(1_000_000)          # an HBM-bound phase: closed
            s.synchronize()
            phases += 1
            if C.ckpt_test(ctx, sid):
                break
            assert time.perf_counter() - t1 < 60, f"the windowed snapshot made no progress ({phases} phases)"
        C.ckpt_wait(ctx, sid)
        want, _, _ = oracle_image(specs, 0, g["L_star"])
        assert_bytes_equal(C.ckpt_host_view(ctx, 0, copy=True)[0], want, "windowed image of 4096 buckets")
    finally:
        C.ckpt_destroy(ctx)


def test_has_split_places_buckets_in_their_windows(torch, C):
    """Alg 1 SplitParameter in the scheduler (ckpt_has_apply): the first bubble_bytes of the
    image go out only in CKPT_WINDOW_BUBBLE windows (they lead, so a compute window moves
    nothing); the rest in CKPT_WINDOW_COMPUTE or bubble windows (Q26); committed images
    match the oracle."""
    import time
    st = tiny(0, n=9)
    specs, ts = st
    B = 1 << 16
    ctx = make_ctx(C, st, n_slots=0, bucket_bytes=B, flags=C.CKPT_OPT_WINDOWED)
    s = torch.cuda.Stream()
    try:
        C.ckpt_protect(ctx, 1, 0)
        g = C.ckpt_geometry(ctx)
        assert g["L"] > 2 * B
        want, _, _ = oracle_image(specs, 0, g["L_star"])
        C.ckpt_has_apply(ctx, B + 1)                     # rounds up to two whole buckets
        C.ckpt_window(ctx, C.CKPT_WINDOW_COMPUTE, s)     # a compute phase: the bubble part waits
        sid = C.ckpt_snapshot(ctx, 0, s)
        time.sleep(0.3)
        assert not C.ckpt_host_view(ctx, 1, copy=True)[0].any(), "bubble buckets left outside a bubble"
        C.ckpt_window(ctx, C.CKPT_WINDOW_BUBBLE, s)      # a bubble: everything may go
        C.ckpt_wait(ctx, sid)
        assert_bytes_equal(C.ckpt_host_view(ctx, 0, copy=True)[0], want, "image after a bubble")
        C.ckpt_has_apply(ctx, 0)                         # all alongside computation
        C.ckpt_window(ctx, 0, s)                         # an HBM-bound phase: closed
        sid = C.ckpt_snapshot(ctx, 0, s)
        time.sleep(0.3)
        assert not C.ckpt_host_view(ctx, 1, copy=True)[0].any(), "D2H while every window was closed"
        C.ckpt_window(ctx, C.CKPT_WINDOW_COMPUTE, s)
        C.ckpt_wait(ctx, sid)
        assert_bytes_equal(C.ckpt_host_view(ctx, 0, copy=True)[0], want, "image after a compute window")
        with pytest.raises(C.CkptError):
            C.ckpt_window(ctx, 8, s)
    finally:
        C.ckpt_destroy(ctx)


def test_has_three_layers_place_buckets(torch, C):
    """HAS Layers 1-3 (P.419-425) in the scheduler (ckpt_has_apply_layers): bubble buckets
    move only in bubbles, the next compute_bytes in compute (or bubble) windows, the rest
    also in communication windows (Layer 3, reading Q28); a communication window alone moves
    only Layer-3 buckets, so the image stays incomplete until the other windows open; the
    committed image matches the oracle."""
    import time
    st = tiny(0, n=9)
    specs, ts = st
    B = 1 << 16
    ctx = make_ctx(C, st, n_slots=0, bucket_bytes=B, flags=C.CKPT_OPT_WINDOWED)
    s = torch.cuda.Stream()
    try:
        C.ckpt_protect(ctx, 1, 0)
        g = C.ckpt_geometry(ctx)
        assert g["L"] > 3 * B
        want, _, _ = oracle_image(specs, 0, g["L_star"])
        C.ckpt_has_apply_layers(ctx, B, B)               # bucket 0: L1, bucket 1: L2, rest: L3
        C.ckpt_window(ctx, C.CKPT_WINDOW_COMM, s)        # an all-reduce phase
        sid = C.ckpt_snapshot(ctx, 0, s)
        time.sleep(0.3)
        d = C.ckpt_host_view(ctx, 1, copy=True)[0]
        assert not d[:2 * B].any(), "Layer 1/2 buckets moved in a communication window"
        C.ckpt_window(ctx, C.CKPT_WINDOW_COMPUTE, s)     # buckets leave in image order: bucket 0 still waits
        time.sleep(0.3)
        assert not C.ckpt_host_view(ctx, 1, copy=True)[0][:B].any(), "Layer 1 bucket moved outside a bubble"
        C.ckpt_window(ctx, C.CKPT_WINDOW_BUBBLE, s)
        C.ckpt_wait(ctx, sid)
        assert_bytes_equal(C.ckpt_host_view(ctx, 0, copy=True)[0], want, "image after all three layers")
        C.ckpt_has_apply_layers(ctx, 0, 0)               # everything in Layer 3
        C.ckpt_window(ctx, 0, s)
        sid = C.ckpt_snapshot(ctx, 0, s)
        time.sleep(0.3)
        assert not C.ckpt_host_view(ctx, 1, copy=True)[0].any(), "D2H while every window was closed"
        C.ckpt_window(ctx, C.CKPT_WINDOW_COMM, s)
        C.ckpt_wait(ctx, sid)
        assert_bytes_equal(C.ckpt_host_view(ctx, 0, copy=True)[0], want, "image after a communication window")
    finally:
        C.ckpt_destroy(ctx)


@pytest.mark.parametrize("m,lost", [(2, 0), (4, 1), (5, 4)])
def test_c_program_drill(torch, C, tmp_path, m, lost):
    """examples/drill_from_c.c: snapshot + parity, loss, rebuild and load through the C ABI
    alone (gcc, include/ckpt.h, -lreft_ckpt -lcudart), tensors checked byte for byte."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.dirname(C.LIB_PATH)
    exe = str(tmp_path / "drill")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(root, "include"),
                           "-I", "/usr/local/cuda/include", os.path.join(root, "examples", "drill_from_c.c"),
                           "-L", libdir, "-lreft_ckpt", "-L", "/usr/local/cuda/lib64", "-lcudart",
                           f"-Wl,-rpath,{libdir}:/usr/local/cuda/lib64", "-o", exe])
    r = subprocess.run([exe, str(m), str(lost)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip() == f"ok m={m} lost={lost}"


@pytest.mark.parametrize("knob", ["CKPT_XOR_IMPL=lsu", "CKPT_XOR_IMPL=tma", "CKPT_PACK_WAVES=1", "CKPT_PACK_WAVES=64", "CKPT_XOR_CTAS=296"])
def test_every_tuning_knob_stays_bit_exact(torch, C, knob):
    """Every environment tuning knob (read once per process, hence a subprocess) under the
    group encode and drill parity tests (every m, unit, staging mode and flag set, incl. the
    push encode) and the smoke (snapshot + parity, rebuild, load): bit-exact vs the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    k, v = knob.split("=")
    env = dict(os.environ, **{k: v})
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", os.path.join(root, "tests", "test_gpu_parity.py"),
                        "-k", "group_encode_matches_oracle or group_drill_rebuild_every_rank or push_encode_repeated"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and " passed" in r.stdout, r.stdout[-3000:] + r.stderr[-2000:]
    r = subprocess.run([sys.executable, os.path.join(root, "__graft_entry__.py"), "smoke"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "smoke ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
