"""GPU parity of AOR (include/ckpt_aor.h; PAPER.md P.494-505, Eq 4) against the oracle.

m ZeRO-1 members share cuda:0 (one AOR context each, as the m processes of a node would);
every member holds the complete flat gradient (P.495).  Per step the test
  - draws the gradient on the device (seeded torch generator: harness input),
  - calls ckpt_aor_step on every member, then ckpt_aor_fence on the training stream,
  - overwrites nothing before the fence; applies the owners' own update on the device
    (torch: master.sub_(g * eta) -- two fp32 roundings, reading Q22),
  - advances the oracle's replicas with oracle.aor_update on the host copy of the gradient.
The replicas must equal the oracle's bit for bit, and the owners' device shards."""
import os

import numpy as np
import pytest

import oracle
from gpu_util import need_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    return need_gpu()


@pytest.fixture(scope="module")
def C(torch):
    from paper_2310_12670_b200 import ckpt
    return ckpt


def fresh_key():
    return int.from_bytes(os.urandom(8), "little") | 1


class Group:
    """m AOR members on cuda:0 with ragged shards of one flat parameter space."""

    def __init__(self, torch, C, sizes, bf16=False, chunk=64 << 10, n_slots=0, threads=0, seed=0, key=None,
                 flags=0):
        self.torch, self.C = torch, C
        self.m = len(sizes)
        self.bounds = [0]
        for n in sizes:
            self.bounds.append(self.bounds[-1] + n)
        self.gen = torch.Generator(device="cuda").manual_seed(seed)
        self.masters = [torch.randn(n, device="cuda", generator=self.gen) for n in sizes]
        self.gdtype = torch.bfloat16 if bf16 else torch.float32
        self.grad = torch.empty(self.bounds[-1], device="cuda", dtype=self.gdtype)
        self.key = key or fresh_key()
        self.opt = dict(key=self.key, chunk_bytes=chunk, n_slots=n_slots, threads=threads, flags=flags,
                        grad_dtype=C.CKPT_DTYPE_BF16 if bf16 else C.CKPT_DTYPE_FP32)
        self.ctx = [self.create(j) for j in range(self.m)]
        torch.cuda.synchronize()
        for j in range(self.m):
            C.ckpt_aor_seed(self.ctx[j], 0)
        # the oracle's replicas: member j holds member (j+1) mod m's shard (ring, SPEC S.313)
        self.rep = [self.masters[(j + 1) % self.m].cpu().numpy() for j in range(self.m)]
        self.t = 0

    def create(self, j):
        o = self.C.ckpt_aor_options_default(**self.opt)
        return self.C.ckpt_aor_create(0, o, self.masters[j], self.grad, self.bounds, j)

    def grad_np(self, j):
        g = self.grad[self.bounds[j]:self.bounds[j + 1]]
        if self.gdtype == self.torch.bfloat16:
            return g.view(self.torch.int16).cpu().numpy().view(np.uint16)
        return g.cpu().numpy()

    def step(self, eta, owners_update=True, members=None):
        torch, C = self.torch, self.C
        members = range(self.m) if members is None else members
        self.grad.copy_(torch.randn(self.bounds[-1], device="cuda", generator=self.gen).to(self.gdtype) * 1e-2)
        ids = {j: C.ckpt_aor_step(self.ctx[j], eta) for j in members}
        for j in members:
            C.ckpt_aor_fence(self.ctx[j], ids[j])
        gs = [self.grad_np(j) for j in range(self.m)]        # synchronizes the stream
        for j in members:
            o = (j + 1) % self.m
            self.rep[j] = oracle.aor_update(self.rep[j], gs[o], eta)
        if owners_update:
            for j in range(self.m):
                g = self.grad[self.bounds[j]:self.bounds[j + 1]].float()
                self.masters[j].sub_(g * eta)
        # the next gradient may overwrite this one only after the fences: poison it now
        self.grad.fill_(float("nan"))
        self.t += 1
        return ids

    def check(self, against_masters=True):
        for j in range(self.m):
            got, step, state = self.C.ckpt_aor_view(self.ctx[j])
            assert state == self.C.CKPT_AOR_CLEAN and step == self.t, (j, step, state)
            assert np.array_equal(got.view(np.uint32), self.rep[j].view(np.uint32)), f"member {j} vs oracle"
            if against_masters:
                dev = self.masters[(j + 1) % self.m].cpu().numpy()
                assert np.array_equal(got.view(np.uint32), dev.view(np.uint32)), f"member {j} vs owner's shard"

    def close(self):
        for a in self.ctx:
            if a:
                self.C.ckpt_aor_destroy(a)
        self.ctx = []


@pytest.mark.parametrize("bf16", [False, True])
@pytest.mark.parametrize("n_slots", [0, 2, 3])
def test_aor_replicas_bit_exact(torch, C, bf16, n_slots):
    # ragged shards spanning many 64 KiB chunks plus tails; a tiny one below one chunk
    g = Group(torch, C, [300_007, 1_000, 131_072 + 5], bf16=bf16, n_slots=n_slots)
    try:
        for t, eta in enumerate([1e-3, 0.37, 3e-4, 1.0]):
            g.step(eta)
        g.check()
        st = C.ckpt_aor_get_stats(g.ctx[2])          # holds member 0's 300,007 elements
        esz = 2 if bf16 else 4
        assert st["steps"] == 4 and st["chunks"] == 4 * -(-300_007 * esz // (64 << 10))
        assert st["d2h_bytes"] == 4 * 300_007 * esz + 4 * (131_072 + 5)   # + its seed of member 2
    finally:
        g.close()


def test_aor_queue_depth_before_wait(torch, C):
    # several steps in flight before any wait: chunks of consecutive steps share the ring
    g = Group(torch, C, [200_003, 150_001], n_slots=2, chunk=128 << 10)
    try:
        ids = [g.step(eta)[0] for eta in (0.1, 0.2, 0.3, 0.4, 0.5)]
        assert ids == [1, 2, 3, 4, 5]
        C.ckpt_aor_wait(g.ctx[0], 5)
        g.check()
    finally:
        g.close()


def test_aor_empty_shard_and_single_member(torch, C):
    g = Group(torch, C, [0, 70_000, 5])      # member 2 holds member 0's empty shard
    try:
        g.step(0.5)
        g.step(0.25)
        g.check()
    finally:
        g.close()
    g = Group(torch, C, [99_999])            # m = 1: a host replica of its own shard
    try:
        g.step(0.125)
        g.check()
    finally:
        g.close()


def test_aor_large_chunks_threads(torch, C):
    # 8 MiB chunks over a 48 MiB shard, 1 and 4 host threads
    for threads in (1, 4):
        g = Group(torch, C, [12 << 20, 3], chunk=8 << 20, threads=threads)
        try:
            g.step(1e-3)
            g.step(2e-3)
            g.check()
        finally:
            g.close()


def test_aor_recover_drill(torch, C):
    """Lose member x (device shard + the replica it held), restart its context (persistent
    objects: a replacement process re-attaches), run the recovery protocol, continue."""
    m = 4
    g = Group(torch, C, [100_003, 77_777, 64_000, 1_234], flags=C.CKPT_AOR_PERSIST)
    try:
        for eta in (0.01, 0.02, 0.03):
            g.step(eta)
        x = 2
        g.masters[x].view(torch.int32).fill_(0x7FA5A5A5)
        C.ckpt_aor_forget(g.ctx[x])
        C.ckpt_aor_destroy(g.ctx[x])
        g.ctx[x] = g.create(x)                     # re-attaches its (poisoned) object
        _, _, state = C.ckpt_aor_view(g.ctx[x])
        assert state == C.CKPT_AOR_POISONED
        with pytest.raises(C.CkptError) as e:      # not CLEAN: nothing to step from
            C.ckpt_aor_step(g.ctx[x], 0.1)
        assert e.value.code == C.CKPT_ESTATE
        # the protocol, in member order (one process here: the barriers are trivially met)
        for j in range(m):
            if j != x:
                C.ckpt_aor_view(g.ctx[j], copy=False)
        step = C.ckpt_aor_restore(g.ctx[x])
        assert step == g.t
        C.ckpt_aor_seed(g.ctx[(x + 1) % m], step)
        torch.cuda.synchronize()
        # the oracle's recovery from the same pre-loss state
        lost = [1 if j == x else 0 for j in range(m)]
        ms = [g.masters[j].cpu().numpy() if j != x else np.full(g.masters[j].numel(), np.nan, np.float32)
              for j in range(m)]
        rs = [g.rep[j] if j != x else np.full(g.rep[j].size, np.nan, np.float32) for j in range(m)]
        want_m, want_r = oracle.aor_recover(lost, ms, rs)
        assert np.array_equal(g.masters[x].cpu().numpy().view(np.uint32), want_m[x].view(np.uint32))
        g.rep = want_r
        for eta in (0.04, 0.05):
            g.step(eta)
        g.check()
    finally:
        g.close()
        C.ckpt_aor_unlink(g.key, m)


def test_aor_adjacent_losses_unrecoverable(torch, C):
    g = Group(torch, C, [10_000, 20_000, 30_000])
    try:
        g.step(0.1)
        C.ckpt_aor_forget(g.ctx[0])                # member 0 lost: the replica of member 1 too
        with pytest.raises(C.CkptError) as e:
            C.ckpt_aor_restore(g.ctx[1])           # member 1 lost as well: its holder is 0
        assert e.value.code == C.CKPT_EUNRECOVERABLE
        assert C.ckpt_aor_restore(g.ctx[2]) == 1   # member 2's holder (1) is intact
    finally:
        g.close()


def test_aor_errors(torch, C):
    key = fresh_key()
    master = torch.zeros(1000, device="cuda")
    grad = torch.zeros(2000, device="cuda")
    o = C.ckpt_aor_options_default(key=key)
    for bad in (dict(key=0), dict(chunk_bytes=4096), dict(n_slots=1), dict(grad_dtype=C.CKPT_DTYPE_FP16)):
        with pytest.raises(C.CkptError) as e:
            C.ckpt_aor_create(0, C.ckpt_aor_options_default(**{**dict(key=key), **bad}), master, grad, [0, 1000, 2000], 0)
        assert e.value.code == C.CKPT_EINVAL
    with pytest.raises(C.CkptError):
        C.ckpt_aor_create(0, o, master, grad, [0, 1000, 900], 0)          # decreasing bounds
    with pytest.raises(C.CkptError) as e:
        C.ckpt_aor_create(0, o, master.cpu(), grad, [0, 1000, 2000], 0)   # host pointer
    assert e.value.code == C.CKPT_EINVAL
    a = C.ckpt_aor_create(0, C.ckpt_aor_options_default(key=key, flags=C.CKPT_AOR_PERSIST), master, grad,
                          [0, 1000, 2000], 0)
    try:
        with pytest.raises(C.CkptError) as e:
            C.ckpt_aor_step(a, 0.1)                                       # never seeded
        assert e.value.code == C.CKPT_ESTATE
        with pytest.raises(C.CkptError) as e:                             # same key, another partition
            C.ckpt_aor_create(0, o, master, grad, [0, 1000, 1999], 0)
        assert e.value.code == C.CKPT_EMISMATCH
    finally:
        C.ckpt_aor_destroy(a)
        C.ckpt_aor_unlink(key, 2)
