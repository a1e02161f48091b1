"""Shared helpers of the GPU parity tests (test infrastructure)."""
import os

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


# ---------------------------------------------------------------------------------------
# Exhaustive (unsampled) comparison at full size.  Every byte of a host image (data D_j and
# parity P_j) is compared with the oracle, streamed window by window so no full oracle image
# is ever held: window w covers image bytes [a, b) (a multiple of the stripe (m-1)u, so the
# parity of the window is exactly P_r[a/(m-1) : b/(m-1)], O4 being stripe-local).  Windows
# run on host threads (the oracle's ctypes calls release the GIL).
# ---------------------------------------------------------------------------------------
def oracle_window(nbytes, offs, rank, a, b, seed=synth.SEED):
    """D_rank[a:b]: the oracle's O3 pack (P.369-371) of the tensor pieces that fall in
    image bytes [a, b), from the oracle's own generator copy.  Bytes outside every tensor
    are the zero pad (Q5)."""
    import bisect
    pieces, where = [], []
    t = max(0, bisect.bisect_right(offs, a) - 1)
    while t < len(nbytes) and offs[t] < b:
        lo, hi = max(a, offs[t]), min(b, offs[t] + nbytes[t])
        if lo < hi:
            pieces.append(oracle.fill(seed, rank, t, hi - lo, lo - offs[t]))
            where.append(lo - a)
        t += 1
    return oracle.pack(pieces, where, b - a)


def _threads():
    return max(1, min(int(os.environ.get("FULLCHECK_THREADS", os.cpu_count() or 1)), 64))


def _first_diff(got, want):
    bad = np.nonzero(got != want)[0]
    return f"{bad.size} bytes differ, first at +{bad[0]} (got {got[bad[0]]:#x} want {want[bad[0]]:#x})"


def verify_images_full(all_specs, Lstar, u, views, ranks=None, rebuild_k=None, seed=synth.SEED,
                       window=64 << 20, gen_ranks=None):
    """Compare every byte of the host images in ``views`` (rank -> (data, parity or None)) with
    the oracle.  ``all_specs[j]`` is member j's tensor list (m = len(all_specs)).  For each
    checked rank j: D_j against O3 and, for m >= 2, P_j against O4 (row j).  With
    ``rebuild_k``: the image of rank k is also compared with O6 (the rebuild from the
    oracle's survivor images and parity), which is what the CUDA rebuild computes.
    Returns the number of bytes compared; raises AssertionError on the first window
    that differs.  ``gen_ranks[j]`` is the generator rank of member j's state (default j)."""
    import concurrent.futures as cf
    m = len(all_specs)
    gen = list(range(m)) if gen_ranks is None else list(gen_ranks)
    ranks = sorted(views) if ranks is None else ranks
    nb = [[s.nbytes for s in sp] for sp in all_specs]
    offs = [oracle.layout(x)[0] for x in nb]
    stripe = (m - 1) * u if m > 1 else 1
    W = max(stripe, window // stripe * stripe)
    if m > 1:
        assert Lstar % stripe == 0

    def one(a):
        b = min(a + W, Lstar)
        need_all = m > 1
        Ds = [oracle_window(nb[j], offs[j], gen[j], a, b, seed) if (need_all or j in ranks) else None
              for j in range(m)]
        n = 0
        for j in ranks:
            d, p = views[j]
            got = np.asarray(d[a:b])
            if not np.array_equal(got, Ds[j]):
                raise AssertionError(f"rank {j} data [{a}, {b}): {_first_diff(got, Ds[j])}")
            n += b - a
            if m > 1 and p is not None:
                Pj = oracle.encode(Ds, u, j)
                gp = np.asarray(p[a // (m - 1):b // (m - 1)])
                if not np.array_equal(gp, Pj):
                    raise AssertionError(f"rank {j} parity [{a // (m - 1)}, {b // (m - 1)}): {_first_diff(gp, Pj)}")
                n += gp.size
        if rebuild_k is not None:
            Ps = [oracle.encode(Ds, u, r) if r != rebuild_k else None for r in range(m)]
            Dsv = [Ds[j] if j != rebuild_k else None for j in range(m)]
            lost = [j == rebuild_k for j in range(m)]
            Dk = oracle.rebuild(Dsv, Ps, u, rebuild_k, lost)
            got = np.asarray(views[rebuild_k][0][a:b])
            if not np.array_equal(got, Dk):
                raise AssertionError(f"rebuilt rank {rebuild_k} [{a}, {b}) vs O6: {_first_diff(got, Dk)}")
        return n

    total = 0
    with cf.ThreadPoolExecutor(_threads()) as ex:
        for n in ex.map(one, range(0, Lstar, W)):
            total += n
    return total


def verify_tensors_full(specs, rank, tensors, seed=synth.SEED):
    """Every byte of every device tensor against the oracle's generator (O7 load: the
    restored tensor equals the bytes that were packed).  Returns bytes compared."""
    import concurrent.futures as cf

    def one(t):
        got = tensor_bytes(tensors[t])
        want = oracle.fill(seed, rank, t, specs[t].nbytes)
        if not np.array_equal(got, want):
            raise AssertionError(f"rank {rank} tensor {t} ({specs[t].name}): {_first_diff(got, want)}")
        return got.size

    with cf.ThreadPoolExecutor(min(_threads(), 16)) as ex:
        return sum(ex.map(one, range(len(specs))))
