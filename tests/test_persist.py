"""Persistent in-memory checkpoint across process death (the paper's
tmpfs persistence, P.553-555; SPEC store atomicity S.431, S.448): a process that dies --
after a commit, or in the middle of the next snapshot -- leaves its last COMMITTED image
in /dev/shm; a restarted process with the same arena key re-attaches it and ckpt_load
restores exactly that state.  A group whose member lost its host memory re-forms and
that member is recovered (ARC / AEC) from the others."""
import os
import traceback

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _child(key, m, scheme, phase, q):
    """phase 'write': snapshot v1, mutate, snapshot v2 committed, mutate, start v3, die.
    phase 'crash_mid': snapshot v1 committed, mutate, start v2 and die without waiting."""
    try:
        import torch

        from paper_2310_12670_b200 import ckpt as C
        from synth.gpu import alloc_state, descriptors, fill_state
        import synth
        ctxs, states = [], []
        for j in range(m):
            specs = synth.config_tensors("tiny_6", j)
            ts = alloc_state(specs, "cuda:0", misalign=1)
            fill_state(ts, j)
            o = C.ckpt_options_default(n_slots=0, bucket_bytes=1 << 16, stripe_unit=4096,
                                       flags=C.CKPT_OPT_SHM_ARENA, arena_key=key)
            c = C.ckpt_create(0, o)
            C.ckpt_register(c, descriptors(ts, specs), {"local_rank": j})
            ctxs.append(c)
            states.append(ts)
        if m == 1:
            C.ckpt_protect(ctxs[0], 1, 0)
        else:
            C.protect_local(ctxs, scheme=scheme)

        def snap(wait=True):
            ids = [C.ckpt_snapshot(c) for c in ctxs]
            if wait:
                for c, i in zip(ctxs, ids):
                    C.ckpt_wait(c, i)

        snap()                                   # v1: the generator state
        for j, ts in enumerate(states):
            fill_state(ts, j, seed=21, xor_mode=1)
        if phase == "write":
            snap()                               # v2: generator ^ seed 21
            for j, ts in enumerate(states):
                fill_state(ts, j, seed=22, xor_mode=1)
        snap(wait=False)                         # in flight when the process dies
        q.put(("ok", None))
        q.close()
        q.join_thread()                          # flush the message, then die abruptly
        os._exit(0)
    except Exception:
        q.put(("err", traceback.format_exc()))
        q.close()
        q.join_thread()
        os._exit(1)


def _reader(key, m, scheme, drop_member, q):
    try:
        import torch

        import oracle
        import synth
        from paper_2310_12670_b200 import ckpt as C
        from synth.gpu import alloc_state, descriptors, fill_state
        if drop_member >= 0:  # that member's host memory is gone (hardware loss)
            for b in range(2):
                try:
                    os.unlink(f"/dev/shm/reft-{key:016x}-{drop_member}-{b}")
                except FileNotFoundError:
                    pass
        ctxs, states, specs_all = [], [], []
        for j in range(m):
            specs = synth.config_tensors("tiny_6", j)
            ts = alloc_state(specs, "cuda:0", misalign=1)
            for t in ts:
                t.view(torch.uint8).fill_(0x77)  # fresh process: garbage in the tensors
            o = C.ckpt_options_default(n_slots=0, bucket_bytes=1 << 16, stripe_unit=4096,
                                       flags=C.CKPT_OPT_SHM_ARENA, arena_key=key)
            c = C.ckpt_create(0, o)
            C.ckpt_register(c, descriptors(ts, specs), {"local_rank": j})
            ctxs.append(c)
            states.append(ts)
            specs_all.append(specs)
        if m == 1:
            C.ckpt_protect(ctxs[0], 1, 0)
        else:
            C.protect_local(ctxs, scheme=scheme)
        if drop_member >= 0:
            for c in ctxs:
                C.ckpt_recover(c, 1 << drop_member)
        for c in ctxs:
            C.ckpt_load(c)
        torch.cuda.synchronize()
        res = []
        for j, (ts, specs) in enumerate(zip(states, specs_all)):
            for t, x in enumerate(ts):
                got = x.contiguous().view(torch.uint8).cpu().numpy()
                res.append((j, t, got.tobytes()))
        for c in ctxs:
            C.ckpt_destroy(c)
        q.put(("ok", res))
    except Exception:
        q.put(("err", traceback.format_exc()))


def _run(target, *args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=target, args=(*args, q))
    p.start()
    status, payload = q.get(timeout=240)
    p.join(60)
    assert status == "ok", payload
    return payload


def _expect(m, seeds):
    import oracle
    import synth
    out = {}
    for j in range(m):
        for t, s in enumerate(synth.config_tensors("tiny_6", j)):
            b = oracle.fill(synth.SEED, j, t, s.nbytes)
            for sd in seeds:
                b = b ^ oracle.fill(sd, j, t, s.nbytes)
            out[(j, t)] = b
    return out


@pytest.fixture(scope="module")
def built():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_2310_12670_b200 import build
    build.build()
    return True


@pytest.mark.parametrize("phase,seeds", [("write", [21]), ("crash_mid", [])])
@pytest.mark.parametrize("m,scheme", [(1, 0), (3, 3), (4, 1)])
def test_restart_reattaches_last_committed(built, phase, seeds, m, scheme):
    from paper_2310_12670_b200 import ckpt as C
    key = int.from_bytes(os.urandom(8), "little") | 1
    try:
        _run(_child, key, m, scheme, phase)
        got = _run(_reader, key, m, scheme, -1)
        want = _expect(m, seeds)
        for j, t, b in got:
            assert np.array_equal(np.frombuffer(b, np.uint8), want[(j, t)]), (j, t)
    finally:
        C.ckpt_arena_unlink(key, max(m, 1), 2)


@pytest.mark.parametrize("m,scheme,drop", [(3, 3, 1), (4, 2, 0), (4, 1, 2)])
def test_restart_after_host_memory_loss(built, m, scheme, drop):
    from paper_2310_12670_b200 import ckpt as C
    key = int.from_bytes(os.urandom(8), "little") | 1
    try:
        _run(_child, key, m, scheme, "write")
        got = _run(_reader, key, m, scheme, drop)
        want = _expect(m, [21])
        for j, t, b in got:
            assert np.array_equal(np.frombuffer(b, np.uint8), want[(j, t)]), (j, t)
    finally:
        C.ckpt_arena_unlink(key, m, 2)


# ---------------------------------------------------------------- AOR (f4) ----------------
# The replica objects are shared memory too: after every member's process died, a restarted
# process re-attaches them (same key) and every member restores its optimizer shard from its
# holder's replica -- exactly the owners' state at the replica's step, or, for a replica an
# update was torn in (the process died inside Eq 4), a refusal.
AOR_SIZES = [60_001, 1_234, 200_000]


def _aor_child(key, phase, q):
    try:
        import torch

        from paper_2310_12670_b200 import ckpt as C
        m = len(AOR_SIZES)
        bounds = [0]
        for n in AOR_SIZES:
            bounds.append(bounds[-1] + n)
        gen = torch.Generator(device="cuda").manual_seed(3)
        masters = [torch.randn(n, device="cuda", generator=gen) for n in AOR_SIZES]
        grad = torch.empty(bounds[-1], device="cuda")
        opt = C.ckpt_aor_options_default(key=key, chunk_bytes=64 << 10, flags=C.CKPT_AOR_PERSIST)
        ctx = [C.ckpt_aor_create(0, opt, masters[j], grad, bounds, j) for j in range(m)]
        for a in ctx:
            C.ckpt_aor_seed(a, 0)
        out = {}
        for t in range(1, 4 if phase == "mid" else 3):
            eta = 0.05 * t
            grad.copy_(torch.randn(bounds[-1], device="cuda", generator=gen) * 1e-2)
            ids = [C.ckpt_aor_step(a, eta) for a in ctx]
            for a, s in zip(ctx, ids):
                C.ckpt_aor_fence(a, s)
            for j in range(m):
                masters[j].sub_(grad[bounds[j]:bounds[j + 1]] * eta)
            out[t] = [x.cpu().numpy().tobytes() for x in masters]
            if t <= 2:
                for a, s in zip(ctx, ids):
                    C.ckpt_aor_wait(a, s)
        q.put(("ok", out))
        q.close()
        q.join_thread()
        os._exit(0)                          # no destroy: the objects stay (persistent)
    except Exception:
        q.put(("err", traceback.format_exc()))
        q.close()
        q.join_thread()
        os._exit(1)


def _aor_reader(key, q):
    try:
        import torch

        from paper_2310_12670_b200 import ckpt as C
        m = len(AOR_SIZES)
        bounds = [0]
        for n in AOR_SIZES:
            bounds.append(bounds[-1] + n)
        masters = [torch.full((n,), float("nan"), device="cuda") for n in AOR_SIZES]
        grad = torch.zeros(bounds[-1], device="cuda")
        opt = C.ckpt_aor_options_default(key=key, chunk_bytes=64 << 10, flags=C.CKPT_AOR_PERSIST)
        ctx = [C.ckpt_aor_create(0, opt, masters[j], grad, bounds, j) for j in range(m)]
        res = []
        for j in range(m):
            try:
                step = C.ckpt_aor_restore(ctx[j])
                torch.cuda.synchronize()
                res.append((j, step, masters[j].cpu().numpy().tobytes()))
            except C.CkptError as e:
                held = ctx[(j - 1) % m]
                res.append((j, e.code, C.ckpt_aor_view(held)[2]))
        for a in ctx:
            C.ckpt_aor_destroy(a)
        q.put(("ok", res))
    except Exception:
        q.put(("err", traceback.format_exc()))


@pytest.mark.parametrize("phase", ["clean", "mid"])
def test_aor_replicas_survive_process_death(built, phase):
    from paper_2310_12670_b200 import ckpt as C
    key = int.from_bytes(os.urandom(8), "little") | 1
    try:
        want = _run(_aor_child, key, phase)
        got = _run(_aor_reader, key)
        for j, a, b in got:
            if phase == "clean" or a in (2, 3) and isinstance(b, bytes):
                assert a == 2 if phase == "clean" else a in (2, 3), (j, a)
                assert b == want[a][j], f"member {j}: restored shard differs from the owner's at step {a}"
            else:                             # a torn replica (Eq 4 was running) is refused
                assert a == C.CKPT_EUNRECOVERABLE and b == C.CKPT_AOR_UPDATING, (j, a, b)
    finally:
        C.ckpt_aor_unlink(key, len(AOR_SIZES))
