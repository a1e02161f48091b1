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


def test_reference_arm_prints_the_contract_line():
    """`bench.py --impl reference` (the oracle as the reference arm, no GPU needed): one JSON
    line with the base contract's keys, impl=reference, a cpu_baseline describing the run
    and a zero-copy e2e; under torchrun only rank 0 prints (here: one process)."""
    import json
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--cpu-seconds", "0.5", "--config", "c1_16mb_fp32_m8"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
