"""Shared helpers of the GPU parity tests (test infrastructure)."""
import numpy as np
import pytest

import oracle
import synth


def need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_12670_b200 import build
    build.build()
    return torch


def oracle_tensor_bytes(specs, rank, seed=synth.SEED):
    """Expected bytes of every tensor of a rank: the ORACLE's own generator copy."""
    return [oracle.fill(seed, rank, t, s.nbytes) for t, s in enumerate(specs)]


def oracle_image(specs, rank, Lstar, seed=synth.SEED, align=256):
    tb = oracle_tensor_bytes(specs, rank, seed)
    off, L = oracle.layout([s.nbytes for s in specs], align)
    return oracle.pack(tb, off, Lstar), off, L


def tensor_bytes(t):
    """Raw bytes of a (possibly bf16) device tensor as a numpy uint8 array."""
    import torch
    return t.detach().contiguous().view(torch.uint8).cpu().numpy().reshape(-1)


def assert_bytes_equal(got, want, what):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, f"{what}: shape {got.shape} != {want.shape}"
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"{what}: {bad.size} bytes differ, first at {bad[0]} "
                             f"(got {got[bad[0]]:#x} want {want[bad[0]]:#x})")


def image_slice(specs, rank, off, n, seed=synth.SEED, align=256):
    """Bytes [off, off+n) of rank's packed image, computed from the oracle's layout rule and
    the oracle's generator copy only (for sampled checks at full size)."""
    offs, L = oracle.layout([s.nbytes for s in specs], align)
    out = np.zeros(n, np.uint8)
    import bisect
    t = max(0, bisect.bisect_right(offs, off) - 1)
    while t < len(specs) and offs[t] < off + n:
        lo, hi = max(off, offs[t]), min(off + n, offs[t] + specs[t].nbytes)
        if lo < hi:
            out[lo - off:hi - off] = oracle.fill(seed, rank, t, hi - lo, lo - offs[t])
        t += 1
    return out
