"""CPU tests of the streaming full-image checker (tests/gpu_util.py) the unsampled GPU
parity tests rely on: it must accept the oracle's own images and reject a single flipped
byte anywhere in data, parity or a rebuilt image, with windows that cut through tensors."""
import numpy as np
import pytest

import oracle
import synth
from gpu_util import verify_images_full


def _images(m, u, n=9):
    specs = [synth.config_tensors(f"tiny_{n}", j) for j in range(m)]
    Ls = []
    for sp in specs:
        Ls.append(oracle.layout([s.nbytes for s in sp])[1])
    Lstar, ue = oracle.common_length(Ls, u) if m > 1 else (Ls[0], u)
    Ds = []
    for j, sp in enumerate(specs):
        off, _ = oracle.layout([s.nbytes for s in sp])
        Ds.append(oracle.pack([oracle.fill(synth.SEED, j, t, s.nbytes) for t, s in enumerate(sp)], off, Lstar))
    Ps = oracle.encode_all(Ds, ue) if m > 1 else [None]
    return specs, Lstar, ue, Ds, Ps


@pytest.mark.parametrize("m,u,window", [(1, 64, 1000), (2, 256, 4096), (3, 64, 1 << 20), (4, 16, 960), (5, 128, 512)])
def test_checker_accepts_oracle_images(m, u, window):
    specs, Lstar, ue, Ds, Ps = _images(m, u)
    views = {j: (Ds[j], Ps[j]) for j in range(m)}
    n = verify_images_full(specs, Lstar, ue, views, window=window)
    assert n == m * (Lstar + (Lstar // (m - 1) if m > 1 else 0))


@pytest.mark.parametrize("m,what", [(1, "data"), (3, "data"), (3, "parity"), (4, "parity"), (4, "rebuilt")])
def test_checker_rejects_one_flipped_byte(m, what):
    specs, Lstar, ue, Ds, Ps = _images(m, 64)
    rng = np.random.default_rng(m)
    for trial in range(4):
        D2 = [d.copy() for d in Ds]
        P2 = [p.copy() if p is not None else None for p in Ps]
        j = int(rng.integers(0, m))
        if what == "parity":
            P2[j][int(rng.integers(0, P2[j].size))] ^= 1 << int(rng.integers(0, 8))
        else:
            D2[j][int(rng.integers(0, Lstar))] ^= 1 << int(rng.integers(0, 8))
        views = {x: (D2[x], P2[x]) for x in range(m)}
        with pytest.raises(AssertionError):
            if what == "rebuilt":
                verify_images_full(specs, Lstar, ue, {j: views[j]}, ranks=[j], rebuild_k=j, window=4 * 64 * 3)
            else:
                verify_images_full(specs, Lstar, ue, views, window=4 * 64 * max(m - 1, 1))


def test_checker_uses_generator_rank_mapping():
    specs, Lstar, ue, Ds, Ps = _images(1, 64)
    with pytest.raises(AssertionError):
        verify_images_full(specs, Lstar, ue, {0: (Ds[0], None)}, gen_ranks=[3])
    assert verify_images_full(specs, Lstar, ue, {0: (Ds[0], None)}, gen_ranks=[0]) == Lstar
