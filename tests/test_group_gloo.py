"""World-size-2 gloo test of the N>1 host logic: the handle exchange of IPC groups
(fixed-size blobs all-gathered in rank order) and node-group membership.  CPU only."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_12670_b200 import ckpt as C
        blob = bytes([rank + 1]) * 8 + bytes(C.CKPT_HANDLE_BYTES - 8)
        allb = C.exchange_handles(blob)
        q.put((rank, len(allb), [allb[j * C.CKPT_HANDLE_BYTES] for j in range(world)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_handles_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    from paper_2310_12670_b200 import ckpt as C
    for rank, n, firsts in res:
        assert n == world * C.CKPT_HANDLE_BYTES
        assert firsts == [j + 1 for j in range(world)]


# ------------------------------------------------------------------ AOR protocol ----------
def _aor_worker(rank, world, port, mask, q):
    """aor_group_key agrees on every rank; aor_recover (include/ckpt_aor.h's protocol) runs
    the right call on each rank between matching barriers.  The C calls are replaced by
    recorders (no GPU here): the host logic is what is under test."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np

        from paper_2310_12670_b200 import ckpt as C
        key = C.aor_group_key()
        keys = [None] * world
        dist.all_gather_object(keys, key)
        calls = []
        C.ckpt_aor_view = lambda a, copy=True: (calls.append("view"), (np.zeros(0, np.float32), 7, 1))[1]
        C.ckpt_aor_restore = lambda a, stream=None: (calls.append("restore"), 7)[1]
        C.ckpt_aor_seed = lambda a, step, stream=None: calls.append(f"seed{step}")
        nbar = [0]

        def barrier():
            nbar[0] += 1
            dist.barrier()

        try:
            step = C.aor_recover(0, mask, rank, world, barrier)
        except C.CkptError as e:
            step = e.code
        q.put((rank, len(set(keys)) == 1 and key != 0, calls, nbar[0], step))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mask", [(2, 0b01), (3, 0b010), (3, 0b101)])
def test_aor_recover_protocol_gloo(world, mask):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_aor_worker, args=(r, world, port, mask, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    lost = [(mask >> j) & 1 for j in range(world)]
    adjacent = any(lost[j] and lost[(j - 1) % world] for j in range(world))
    for rank, key_ok, calls, nbar, step in res:
        assert key_ok
        if adjacent:                       # refused on every rank before any call
            assert calls == [] and nbar == 0 and step == -10
            continue
        want = ["restore"] if lost[rank] else ["view"]
        if not lost[rank] and lost[(rank - 1) % world]:
            want.append("seed7")           # re-creates the replica its lost holder kept
        assert calls == want, (rank, calls)
        assert nbar == 3 and step == 7
