"""Build the in-tree CUDA libraries for sm_100a with nvcc (no JIT, no torch ext).

  libreft_ckpt.so  -- the product: C ABI of include/ckpt.h and include/ckpt_aor.h
  libreft_synth.so -- harness: seeded GPU generator of include/reft_synth.h

Both link the CUDA runtime statically; the driver API entry points (stream memory
operations) are resolved at run time with cudaGetDriverEntryPoint.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-Wall,-fvisibility=hidden,-ffp-contract=off", "-shared",
         "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include")]

LIBS = {
    "libreft_ckpt.so": ["ckpt_api.cu", "ckpt_hostmem.cu", "ckpt_pipeline.cu", "ckpt_recovery.cu", "ckpt_kernels.cu", "ckpt_probe.cu",
                        "ckpt_aor.cu", "aor_update.cpp"],
    "libreft_synth.so": ["synth_fill.cu"],
}


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = srcs + [os.path.join(CSRC, "ckpt_kernels.cuh"), os.path.join(CSRC, "ckpt_internal.cuh"),
                   os.path.join(ROOT, "include", "ckpt.h"), os.path.join(ROOT, "include", "ckpt_aor.h"),
                   os.path.join(ROOT, "include", "reft_synth.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> dict:
    out = {}
    for lib, srcs in LIBS.items():
        path = os.path.join(HERE, lib)
        srcs = [os.path.join(CSRC, s) for s in srcs]
        if force or _stale(path, srcs):
            tmp = path + f".tmp{os.getpid()}"
            cmd = [NVCC, *ARCH, *FLAGS, "-o", tmp, *srcs]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed for {lib}")
            if verbose:
                sys.stderr.write(r.stderr)
            os.replace(tmp, path)
            with open(os.path.join(HERE, lib + ".ptxas.txt"), "w") as f:
                f.write(r.stderr)
        out[lib] = path
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
