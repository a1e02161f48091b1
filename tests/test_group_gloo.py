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
