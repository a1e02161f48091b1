"""CPU oracle for REFT snapshot-and-protect -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Thin ctypes wrapper over ``oracle/reft_oracle.c`` (plain scalar byte loops).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  It shares no code with the
CUDA path (``paper_2310_12670_b200``) and imports nothing from it.

Functions follow SURVEY.md 8(c) O1-O7; each C function cites the paper passage
(Eq 1 P.474-477, Eq 2 P.481-484, sub-slicing P.486, load P.545).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "reft_oracle.c")
_LIB = os.path.join(_HERE, "libreft_oracle.so")

EINVAL = -1
EUNRECOVERABLE = -2

_u64 = ctypes.c_uint64
_p = ctypes.c_void_p
_lib = None


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, no tuning flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.oracle_layout.argtypes = [_u64, _p, _u64, _p, _p]
        L.oracle_common_length.argtypes = [_u64, _p, _u64, _p, _p]
        L.oracle_pack.argtypes = [_u64, _p, _p, _p, _u64, _p]
        L.oracle_unpack.argtypes = [_u64, _p, _p, _p, _u64, _p]
        L.oracle_encode.argtypes = [_u64, _p, _u64, _u64, _u64, _p]
        L.oracle_rebuild.argtypes = [_u64, _p, _p, _u64, _u64, _u64, _p, _p]
        L.oracle_fill.argtypes = [_u64, _u64, _u64, _u64, _u64, _p]
        L.oracle_arc_holder.argtypes = [_u64, _u64]
        L.oracle_arc_holder.restype = _u64
        L.oracle_arc_copy.argtypes = [_u64, _p, _u64, _u64, _p]
        L.oracle_recover.argtypes = [_u64, _u64, _p, _p, _p, _p, _p, _u64, _u64, _p, _p]
        L.oracle_aor_update.argtypes = [_u64, _p, _p, _u64, ctypes.c_float]
        L.oracle_aor_recover.argtypes = [_u64, _p, _p, _p, _p]
        L.oracle_splitmix64.argtypes = [_u64]
        L.oracle_splitmix64.restype = _u64
        for f in ("oracle_layout", "oracle_common_length", "oracle_pack", "oracle_unpack",
                  "oracle_encode", "oracle_rebuild", "oracle_fill", "oracle_arc_copy", "oracle_recover",
                  "oracle_aor_update", "oracle_aor_recover"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _chk(rc: int, what: str) -> None:
    if rc == EUNRECOVERABLE:
        raise OracleError(f"{what}: unrecoverable")
    if rc != 0:
        raise OracleError(f"{what}: rc={rc}")


def _u64arr(xs) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(xs, dtype=np.uint64))


def _ptrs(bufs) -> np.ndarray:
    return np.array([b.ctypes.data if b is not None else 0 for b in bufs], dtype=np.uint64)


def _bytes(a) -> np.ndarray:
    a = np.ascontiguousarray(a)
    return a.view(np.uint8).reshape(-1)


# ---- O1 / O2 -----------------------------------------------------------------
def layout(nbytes, align: int = 256):
    """O1: offsets of each tensor in the packed image and the rank's length L_j."""
    nb = _u64arr(nbytes)
    off = np.zeros(max(len(nb), 1), dtype=np.uint64)
    L = np.zeros(1, dtype=np.uint64)
    _chk(lib().oracle_layout(len(nb), nb.ctypes.data, align, off.ctypes.data, L.ctypes.data), "layout")
    return off[: len(nb)].astype(np.int64).tolist(), int(L[0])


def common_length(Ls, u: int):
    """O2: (L*, u_eff) for a group whose members have packed lengths ``Ls``."""
    Lj = _u64arr(Ls)
    Ls_ = np.zeros(1, dtype=np.uint64)
    ue = np.zeros(1, dtype=np.uint64)
    _chk(lib().oracle_common_length(len(Lj), Lj.ctypes.data, u, Ls_.ctypes.data, ue.ctypes.data),
         "common_length")
    return int(Ls_[0]), int(ue[0])


# ---- O3 / O7 -----------------------------------------------------------------
def pack(tensors, offsets, Lstar: int) -> np.ndarray:
    """O3: packed image D (uint8[L*]) of a list of byte arrays."""
    srcs = [_bytes(t) for t in tensors]
    nb = _u64arr([s.size for s in srcs])
    off = _u64arr(offsets)
    D = np.empty(Lstar, dtype=np.uint8)
    ptr = _ptrs(srcs)
    _chk(lib().oracle_pack(len(srcs), ptr.ctypes.data, nb.ctypes.data, off.ctypes.data, Lstar,
                           D.ctypes.data), "pack")
    return D


def unpack(D: np.ndarray, nbytes, offsets):
    """O7: list of uint8 arrays restored from image D."""
    outs = [np.empty(int(n), dtype=np.uint8) for n in nbytes]
    nb = _u64arr(nbytes)
    off = _u64arr(offsets)
    ptr = _ptrs(outs)
    D = np.ascontiguousarray(D, dtype=np.uint8)
    _chk(lib().oracle_unpack(len(outs), ptr.ctypes.data, nb.ctypes.data, off.ctypes.data, D.size,
                             D.ctypes.data), "unpack")
    return outs


# ---- O4 / O6 -----------------------------------------------------------------
def encode(Ds, u: int, r: int) -> np.ndarray:
    """O4: parity stream of row-holder r (uint8[L*/(m-1)]) from the m packed images."""
    m = len(Ds)
    Ds = [np.ascontiguousarray(d, dtype=np.uint8) for d in Ds]
    Lstar = Ds[0].size
    P = np.empty(Lstar // max(m - 1, 1), dtype=np.uint8)
    ptr = _ptrs(Ds)
    _chk(lib().oracle_encode(m, ptr.ctypes.data, Lstar, u, r, P.ctypes.data), "encode")
    return P


def encode_all(Ds, u: int):
    return [encode(Ds, u, r) for r in range(len(Ds))]


def rebuild(Ds, Ps, u: int, k: int, lost=None) -> np.ndarray:
    """O6: rank k's packed image from the survivors' images and parity streams.
    ``Ds[k]``/``Ps[k]`` may be None (they are never read)."""
    m = len(Ds)
    Lstar = next(d.size for d in Ds if d is not None)
    Dk = np.empty(Lstar, dtype=np.uint8)
    Ds_ = [np.ascontiguousarray(d, dtype=np.uint8) if d is not None else None for d in Ds]
    Ps_ = [np.ascontiguousarray(p, dtype=np.uint8) if p is not None else None for p in Ps]
    lost_arr = None
    if lost is not None:
        lost_arr = np.array([1 if x else 0 for x in lost], dtype=np.uint8)
    dptr, pptr = _ptrs(Ds_), _ptrs(Ps_)
    _chk(lib().oracle_rebuild(m, dptr.ctypes.data, pptr.ctypes.data, Lstar, u, k,
                              lost_arr.ctypes.data if lost_arr is not None else None,
                              Dk.ctypes.data), "rebuild")
    return Dk


# ---- ARC / collaborative protection -----------------------------
SCHEME_AEC, SCHEME_ARC, SCHEME_ARC_AEC = 1, 2, 3


def arc_holder(m: int, x: int) -> int:
    """Member holding the ARC copy of member x (ring placement, SPEC S.313)."""
    return int(lib().oracle_arc_holder(m, x))


def arc_copy(Ds, i: int) -> np.ndarray:
    """ARC copy held by member i: the image of member (i+1) mod m."""
    Ds = [np.ascontiguousarray(d, dtype=np.uint8) for d in Ds]
    out = np.empty(Ds[0].size, dtype=np.uint8)
    ptr = _ptrs(Ds)
    _chk(lib().oracle_arc_copy(len(Ds), ptr.ctypes.data, Ds[0].size, i, out.ctypes.data), "arc_copy")
    return out


def recover(scheme: int, lost, Ds, Ps, MDs, MPs, u: int):
    """REFT-load step 3 for up to two losses; returns {x: (D_x, P_x or None)}.
    Entries of lost members in Ds/Ps/MDs/MPs may be None (never read)."""
    m = len(Ds)
    sizes = [d.size for d in list(Ds) + list(MDs or []) if d is not None]
    if not sizes:
        raise OracleError("recover: unrecoverable (no surviving member)")
    Lstar = sizes[0]
    pb = Lstar // max(m - 1, 1)
    aec = scheme in (SCHEME_AEC, SCHEME_ARC_AEC)
    lost_arr = np.array([1 if x else 0 for x in lost], dtype=np.uint8)
    outD = [np.zeros(Lstar, np.uint8) if lost[j] else None for j in range(m)]
    outP = [np.zeros(pb, np.uint8) if lost[j] and aec else None for j in range(m)]
    keep = [[np.ascontiguousarray(a, dtype=np.uint8) if a is not None else None for a in arr]
            for arr in (Ds, Ps or [None] * m, MDs or [None] * m, MPs or [None] * m)]
    ptrs = [_ptrs(k) for k in keep]
    po, pp = _ptrs(outD), _ptrs(outP)
    _chk(lib().oracle_recover(m, scheme, lost_arr.ctypes.data, ptrs[0].ctypes.data, ptrs[1].ctypes.data,
                              ptrs[2].ctypes.data, ptrs[3].ctypes.data, Lstar, u, po.ctypes.data, pp.ctypes.data),
         "recover")
    return {j: (outD[j], outP[j]) for j in range(m) if lost[j]}


# ---- AOR (Eq 4, P.494-505) -------------------------------
DTYPE_BF16, DTYPE_FP32 = 1, 3


def aor_update(w: np.ndarray, grad: np.ndarray, eta: float) -> np.ndarray:
    """One Eq 4 step on a copy of replica ``w`` (float32): w - fp32(eta * g).
    ``grad`` is float32, or uint16 holding bf16 bits."""
    out = np.array(w, dtype=np.float32, copy=True)
    g = np.ascontiguousarray(grad)
    if g.dtype == np.float32:
        dt = DTYPE_FP32
    elif g.dtype == np.uint16:
        dt = DTYPE_BF16
    else:
        raise OracleError("aor_update: grad must be float32 or uint16 (bf16 bits)")
    if g.size != out.size:
        raise OracleError("aor_update: size mismatch")
    _chk(lib().oracle_aor_update(out.size, out.ctypes.data, g.ctypes.data, dt, ctypes.c_float(eta)), "aor_update")
    return out


def aor_recover(lost, masters, replicas):
    """AOR recovery (P.505): returns (masters, replicas) after restoring the lost members.
    ``replicas[j]`` is the replica member j holds of member (j+1) mod m."""
    m = len(masters)
    ms = [np.array(x, dtype=np.float32, copy=True) for x in masters]
    rs = [np.array(x, dtype=np.float32, copy=True) for x in replicas]
    lost_arr = np.array([1 if x else 0 for x in lost], dtype=np.uint8)
    n = _u64arr([x.size for x in ms])
    pm, pr = _ptrs(ms), _ptrs(rs)   # keep the pointer arrays alive across the call
    _chk(lib().oracle_aor_recover(m, lost_arr.ctypes.data, pm.ctypes.data, pr.ctypes.data, n.ctypes.data),
         "aor_recover")
    return ms, rs


# ---- generator (oracle's own copy; not part of the method) ------------------------
def splitmix64(x: int) -> int:
    return int(lib().oracle_splitmix64(x))


def fill(seed: int, rank: int, tensor: int, nbytes: int, byte_begin: int = 0) -> np.ndarray:
    out = np.empty(nbytes, dtype=np.uint8)
    _chk(lib().oracle_fill(seed, rank, tensor, byte_begin, nbytes, out.ctypes.data), "fill")
    return out
