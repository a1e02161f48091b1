"""CPU checks of bench.py's baseline legs (no GPU): the all-cores oracle timing
(`OracleGroup`, `cpu_baseline.all_cores` / `parity_all_cores_m4` and the `--impl reference`
arm) cuts every member's image into stripe-aligned windows, one per host thread, and runs
the unchanged oracle on each.  Its claim -- that a window's pack, parity rows and rebuild
are exactly the corresponding slices of the whole-image results (O3/O4/O6 are stripe-local)
-- is checked here against the oracle on whole images."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("m,unit,threads", [(1, 4096, 3), (2, 4096, 2), (3, 1024, 4), (4, 16384, 2)])
def test_oracle_group_windows_are_slices_of_the_whole_image(m, unit, threads):
    import bench
    import oracle
    import synth

    og = bench.OracleGroup("tiny_40", m, 0.01, threads, unit)
    og.run(keep=True)
    W = og.W
    stripe = (m - 1) * unit if m > 1 else 65536
    assert W % stripe == 0 and W > 0
    specs = [synth.config_tensors("tiny_40", j) for j in range(m)]
    imgs = []
    for j, sp in enumerate(specs):
        off, L = oracle.layout([s.nbytes for s in sp])
        tb = [synth.fill(synth.SEED, j, t, s.nbytes) for t, s in enumerate(sp)]
        imgs.append(oracle.pack(tb, off, max(L, threads * W)))   # zero beyond L, like the windows
    if m > 1:
        Ls, u = oracle.common_length([x.size for x in imgs], unit)
        imgs = [np.concatenate([d, np.zeros(max(0, Ls - d.size), np.uint8)]) for d in imgs]
        Ps = [oracle.encode(imgs, u, r) for r in range(m)]
    for i in range(threads):
        Ds, Pw, R = og.out[i]
        a, b = i * W, (i + 1) * W
        for j in range(m):
            assert np.array_equal(Ds[j], imgs[j][a:b]), f"window {i} member {j} image"
        if m > 1:
            for r in range(m):
                assert np.array_equal(Pw[r], Ps[r][a // (m - 1):b // (m - 1)]), f"window {i} parity row {r}"
            assert np.array_equal(R, imgs[0][a:b]), f"window {i} rebuild of member 0"
