"""CPU-only checks of the C ABI library: it builds, loads, exports every symbol
include/*.h declares, its host-only planner agrees with the oracle's layout pins, and
it refuses to run without a GPU (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT, golden


@pytest.fixture(scope="module")
def C():
    from paper_2310_12670_b200 import build, ckpt
    build.build()
    return ckpt


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:ckpt|reft)_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(C):
    import ctypes
    lib = ctypes.CDLL(C.LIB_PATH)
    names = declared("ckpt.h")
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"libreft_ckpt.so does not export {n}"
    aor = declared("ckpt_aor.h")
    assert len(aor) >= 12
    for n in aor:
        assert hasattr(lib, n), f"libreft_ckpt.so does not export {n}"
    synth = ctypes.CDLL(C.SYNTH_PATH)
    for n in declared("reft_synth.h"):
        assert hasattr(synth, n), n


def test_library_is_sm100a():
    import subprocess
    from paper_2310_12670_b200 import build
    libs = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libs["libreft_ckpt.so"]],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", libs["libreft_ckpt.so"]],
                          capture_output=True, text=True).stdout
    assert "UBLKCP" in sass          # TMA 1-D bulk copies in the TMA pack kernel
    assert "LDG.E.128" in sass       # 128-bit loads in the LSU pack / XOR kernels


def test_plan_layout_matches_oracle_golden(C):
    g = golden("layout_a256.txt")
    sizes = [int(x) for x in g["sizes"][0]]
    assert C.ckpt_plan_layout(sizes, 256) == oracle.layout(sizes, 256)
    assert C.ckpt_plan_layout(sizes, 256)[0] == [int(x) for x in g["offsets"][0]]
    for m, u, Ls, ue in g["common"]:
        assert C.ckpt_plan_common([1280, 768, 1024][: int(m)], int(u)) == (int(Ls), int(ue))


def test_plan_random_vs_oracle(C):
    rng = np.random.default_rng(5)
    for _ in range(200):
        sizes = rng.integers(1, 1 << 20, size=int(rng.integers(1, 30))).tolist()
        align = int(2 ** rng.integers(4, 13))
        assert C.ckpt_plan_layout(sizes, align) == oracle.layout(sizes, align)
        m = int(rng.integers(1, 9))
        Ls = rng.integers(1, 1 << 24, size=m).tolist()
        u = int(rng.choice([0, 16, 4096, 65536, 1 << 20]))  # 1 MiB: the default since round 2
        assert C.ckpt_plan_common(Ls, u) == oracle.common_length(Ls, u)


def test_no_gpu_means_error_not_fallback(C):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(C.CkptError) as e:
        C.ckpt_create(0)
    assert e.value.code == C.CKPT_ECUDA
    assert "no CPU fallback" in str(e.value)


def test_strerror_and_version(C):
    assert C.ckpt_strerror(C.CKPT_EUNRECOVERABLE).startswith("unrecoverable")
    assert C.ckpt_strerror(12345) == "unknown error"
    assert "sm_100a" in C.ckpt_version()


def test_options_defaults(C):
    o = C.ckpt_options_default()
    assert (o.align, o.stripe_unit, o.bucket_bytes, o.n_slots, o.host_buffers) == (256, 1 << 20, 64 << 20, 4, 2)


def test_has_plan_spec_vectors(C):
    """Alg 1 (P.377-413) estimators against SPEC's worked examples (S.185-187, S.242-248,
    S.236): EstimateBubbleTime(p=0,|P|=4,C=1) = 6.0; (p=3,|P|=4,C=2) = 10.8; |P|=1 -> 0;
    EstimateSnapshotTime(16 GiB at 16 GiB/s) = 1.0 s; SplitParameter(100, t_ss=10,
    t_bubble=4) = (40, 60); t_ss < t_bubble -> (100, 0); t_bubble = 0 -> (0, 100)."""
    assert C.ckpt_has_plan(0, 4, 1.0, 1, 1.0)["t_bubble"] == pytest.approx(6.0)
    assert C.ckpt_has_plan(3, 4, 2.0, 1, 1.0)["t_bubble"] == pytest.approx(10.8)
    assert C.ckpt_has_plan(0, 1, 5.0, 1, 1.0)["t_bubble"] == 0.0
    assert C.ckpt_has_plan(0, 1, 1.0, 16 << 30, float(16 << 30))["t_ss"] == pytest.approx(1.0)
    p = C.ckpt_has_plan(0, 3, 1.0, 100, 10.0)  # t_bubble = (2*3-2)*1 = 4, t_ss = 100/10 = 10
    assert (p["t_ss"], p["t_bubble"], p["bubble_bytes"], p["compute_bytes"]) == (10.0, 4.0, 40, 60)
    p = C.ckpt_has_plan(0, 6, 1.0, 100, 20.0)  # t_bubble 10 > t_ss 5
    assert (p["bubble_bytes"], p["compute_bytes"]) == (100, 0)
    p = C.ckpt_has_plan(0, 1, 1.0, 100, 10.0)  # no pipeline, no bubble
    assert (p["bubble_bytes"], p["compute_bytes"]) == (0, 100)
    with pytest.raises(C.CkptError):
        C.ckpt_has_plan(4, 4, 1.0, 1, 1.0)


def test_has_plan3_layers(C):
    """HAS Layers 1-3 (P.419-425, reading Q28): Layer 1 is Alg 1's W_bubble unchanged; Layer 2
    takes floor(n * t_compute / t_ss) of the rest; Layer 3 only what the first two cannot
    hold ("not used unless the previous layers are not enough"); the three partition n."""
    # n = 100, t_ss = 10, t_bubble = 4 (p=0, |P|=3, C=1): W_bubble = 40 as in Alg 1
    p = C.ckpt_has_plan3(0, 3, 1.0, 100, 10.0, 3.0)   # compute holds 30 of the remaining 60
    assert (p["bubble_bytes"], p["compute_bytes"], p["comm_bytes"]) == (40, 30, 30)
    p = C.ckpt_has_plan3(0, 3, 1.0, 100, 10.0, 6.0)   # compute holds all 60: no Layer 3
    assert (p["bubble_bytes"], p["compute_bytes"], p["comm_bytes"]) == (40, 60, 0)
    p = C.ckpt_has_plan3(0, 3, 1.0, 100, 10.0, 0.0)   # no compute window: the rest is Layer 3
    assert (p["bubble_bytes"], p["compute_bytes"], p["comm_bytes"]) == (40, 0, 60)
    p = C.ckpt_has_plan3(0, 6, 1.0, 100, 20.0, 0.0)   # bubbles hold everything
    assert (p["bubble_bytes"], p["compute_bytes"], p["comm_bytes"]) == (100, 0, 0)
    for args in [(0, 4, 0.7, 12345, 3.0, 1.1), (2, 4, 0.3, 10 ** 9, 7.0, 0.05), (0, 1, 1.0, 999, 1.0, 0.5)]:
        p = C.ckpt_has_plan3(*args)
        q = C.ckpt_has_plan(*args[:5])
        assert p["bubble_bytes"] == q["bubble_bytes"]
        assert p["bubble_bytes"] + p["compute_bytes"] + p["comm_bytes"] == args[3]
    with pytest.raises(C.CkptError):
        C.ckpt_has_plan3(0, 3, 1.0, 100, 10.0, -1.0)


# ---------------------------------------------------------------- AOR host arithmetic ----
@pytest.mark.parametrize("bf16", [False, True])
def test_aor_host_update_matches_oracle(C, bf16):
    """The library's Eq 4 routine (the one its worker threads run) vs the oracle, bit for bit,
    over ragged lengths that exercise the AVX-512 body and the scalar tail."""
    rng = np.random.default_rng(11)
    for n in (0, 1, 15, 16, 17, 31, 33, 1000, 65_537):
        w = rng.standard_normal(n).astype(np.float32)
        if bf16:
            g = (rng.standard_normal(n).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
        else:
            g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
        for eta in (1e-3, 0.37, 1.0):
            got = w.copy()
            C.ckpt_aor_apply(got, g, eta)
            assert np.array_equal(got.view(np.uint32), oracle.aor_update(w, g, eta).view(np.uint32)), (n, eta)


def test_aor_host_update_has_no_fma():
    """Reading Q22 (product rounded before the subtraction): no fused multiply-add in the
    library's host update routines (build.py passes -ffp-contract=off)."""
    import subprocess
    from paper_2310_12670_b200 import build
    so = build.build()["libreft_ckpt.so"]
    dis = subprocess.run(["objdump", "-d", "--no-show-raw-insn", so], capture_output=True, text=True).stdout
    body, cur = {}, None
    for line in dis.splitlines():
        if line.endswith(">:"):
            cur = line if "sgd" in line else None
            if cur:
                body[cur] = []
        elif not line.strip():
            cur = None
        elif cur:
            body[cur].append(line)
    assert len(body) >= 3 and any("aor_sgd" in k for k in body), "update routines not found"
    insns = "\n".join("\n".join(v) for v in body.values())
    assert "vmulps" in insns and "vsubps" in insns
    assert not re.search(r"\bv?f(n)?m(add|sub)", insns), "FMA found in the Eq 4 routines"


def test_aor_no_gpu_means_error(C):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    o = C.ckpt_aor_options_default(key=12345)
    with pytest.raises(C.CkptError) as e:
        C.ckpt_aor_create(0, o, 0x1000, 0x2000, [0, 10, 20], 0)
    assert e.value.code == C.CKPT_ECUDA


def test_aor_options_and_protocol_guard(C):
    o = C.ckpt_aor_options_default()
    assert (o.grad_dtype, o.chunk_bytes, o.n_slots, o.key) == (C.CKPT_DTYPE_FP32, 16 << 20, 0, 0)
    # adjacent losses are refused before any barrier or call (oracle_aor_recover's rule)
    with pytest.raises(C.CkptError) as e:
        C.aor_recover(0, 0b0110, 1, 4, barrier=lambda: None)
    assert e.value.code == C.CKPT_EUNRECOVERABLE


def test_c_program_uses_the_abi(C, tmp_path):
    """examples/plan_from_c.c: the library from plain C (gcc, include/*.h, -lreft_ckpt), its
    host-only results checked against the oracle and the Q22 closed form."""
    import struct
    import subprocess
    libdir = os.path.dirname(C.LIB_PATH)
    exe = str(tmp_path / "plan_from_c")
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "examples", "plan_from_c.c"), "-L", libdir, "-lreft_ckpt",
                           f"-Wl,-rpath,{libdir}", "-o", exe])
    out = dict(line.split(" ", 1) for line in subprocess.check_output([exe], text=True).splitlines())
    off, L = oracle.layout([1000, 4096, 1, 70000, 255], 256)
    assert out["layout"] == f"rc=0 L={L} off={','.join(map(str, off))}"
    Ls, ue = oracle.common_length([L, 1280, 99840], 4096)
    assert out["common"] == f"rc=0 Lstar={Ls} unit={ue}"
    assert out["has"] == "rc=0 t_ss=10.000 t_bubble=4.000 bubble=40 compute=60"
    want = [struct.unpack("<I", struct.pack("<f", x))[0] for x in (1.0 - 0.125, -3.5 + 0.0625, 1024.0 - 2.0)]
    assert out["aor"] == "rc=0 w=" + ",".join(f"{x:08x}" for x in want)
    assert out["bad"].startswith("rc=-1 (invalid argument)")
    assert "sm_100a" in out["version"]


def test_scripts_compile():
    """bench.py, __graft_entry__.py and every tool parse (they run only on GPU boxes)."""
    import ast
    import glob
    files = [os.path.join(ROOT, "bench.py"), os.path.join(ROOT, "__graft_entry__.py")] + \
        sorted(glob.glob(os.path.join(ROOT, "tools", "*.py")))
    for f in files:
        ast.parse(open(f).read(), filename=f)
