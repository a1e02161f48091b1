"""Thin ctypes binding of libreft_ckpt (include/ckpt.h): same names, argument
marshalling only.  Every step of the hot path runs in the CUDA library; there is no
CPU fallback -- importing this module on a machine without the built library raises.

PyTorch is used only as plumbing: device tensors (their data pointers), CUDA streams
(their handles) and ``torch.distributed`` for the handle exchange of IPC groups.
"""
from __future__ import annotations

import ctypes
import os
from typing import Iterable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libreft_ckpt.so")
SYNTH_PATH = os.path.join(_HERE, "libreft_synth.so")

CKPT_OK = 0
CKPT_EINVAL = -1
CKPT_ECUDA = -2
CKPT_ENOMEM = -3
CKPT_ESTATE = -4
CKPT_EUNAVAIL = -5
CKPT_EMISMATCH = -6
CKPT_EPEER = -7
CKPT_EBUSY = -8
CKPT_ENOSNAP = -9
CKPT_EUNRECOVERABLE = -10

CKPT_OPT_TIMING = 0x1
CKPT_OPT_TMA_PACK = 0x2
CKPT_OPT_LSU_PACK = 0x4
CKPT_OPT_CE_PACK = 0x8
CKPT_OPT_CE_GATHER = 0x10
CKPT_OPT_DEVICE_ONLY = 0x20
CKPT_OPT_SHM_ARENA = 0x40
CKPT_OPT_HOST_LOAD = 0x80
CKPT_OPT_WINDOWED = 0x100
CKPT_OPT_REBUILD_SHARES = 0x200
CKPT_OPT_REBUILD_SELF = 0x800
CKPT_OPT_XOR_PUSH = 0x400
CKPT_PROBE_SM_PULL, CKPT_PROBE_CE_PULL = 0, 1
CKPT_SCHEME_DEFAULT, CKPT_SCHEME_AEC, CKPT_SCHEME_ARC, CKPT_SCHEME_ARC_AEC = 0, 1, 2, 3

CKPT_DTYPE_BYTES, CKPT_DTYPE_BF16, CKPT_DTYPE_FP16, CKPT_DTYPE_FP32 = 0, 1, 2, 3
CKPT_ROLE_PARAM, CKPT_ROLE_MASTER, CKPT_ROLE_EXP_AVG, CKPT_ROLE_EXP_AVG_SQ, CKPT_ROLE_OTHER = 0, 1, 2, 3, 4
CKPT_TENSOR_REPLICATED = 0x1

CKPT_HANDLE_BYTES = 1024
CKPT_MAX_GROUP = 8
CKPT_GROUP_IPC = 0
CKPT_GROUP_LOCAL = 1

_u32, _u64, _i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32
_vp = ctypes.c_void_p


class ckpt_options(ctypes.Structure):
    _fields_ = [("struct_size", _u32), ("align", _u32), ("stripe_unit", _u64), ("bucket_bytes", _u64),
                ("n_slots", _u32), ("host_buffers", _u32), ("priority", _i32), ("max_ctas", _u32),
                ("flags", _u32), ("reserved0", _u32), ("arena_key", _u64), ("reserved", _u32 * 4)]


class ckpt_tensor(ctypes.Structure):
    _fields_ = [("dev_ptr", _vp), ("nbytes", _u64), ("dtype", _u32), ("role", _u32), ("flags", _u32),
                ("reserved", _u32), ("name", ctypes.c_char_p)]


class ckpt_layout(ctypes.Structure):
    _fields_ = [(n, _i32) for n in ("rank", "world", "local_rank", "local_world", "tp_rank", "tp_size",
                                    "pp_rank", "pp_size", "dp_rank", "dp_size")]


class ckpt_group(ctypes.Structure):
    _fields_ = [("m", _u32), ("my_index", _u32), ("transport", _u32), ("scheme", _u32),
                ("handles", _vp), ("members", ctypes.POINTER(_vp))]


class ckpt_stats(ctypes.Structure):
    _fields_ = [(n, _u64) for n in ("snapshots", "loads", "rebuilds", "pack_launches", "xor_launches",
                                    "unpack_launches", "rebuild_launches", "pack_bytes", "xor_bytes_in",
                                    "xor_bytes_out", "d2h_bytes", "h2d_bytes", "ce_copies", "rebuild_bytes_in",
                                    "rebuild_bytes_out")] + \
               [(n, ctypes.c_double) for n in ("pack_ms", "xor_ms", "unpack_ms", "rebuild_ms", "last_snapshot_ms")] + \
               [("gather_ops", _u64), ("gather_ms", ctypes.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class ckpt_has_plan_t(ctypes.Structure):
    _fields_ = [("t_ss", ctypes.c_double), ("t_bubble", ctypes.c_double), ("bubble_bytes", _u64),
                ("compute_bytes", _u64)]


class ckpt_has_plan3_t(ctypes.Structure):
    _fields_ = [("t_ss", ctypes.c_double), ("t_bubble", ctypes.c_double), ("t_compute", ctypes.c_double),
                ("bubble_bytes", _u64), ("compute_bytes", _u64), ("comm_bytes", _u64)]


CKPT_AOR_PERSIST = 0x1
CKPT_AOR_EMPTY, CKPT_AOR_CLEAN, CKPT_AOR_UPDATING, CKPT_AOR_POISONED, CKPT_AOR_SEEDING = 0, 1, 2, 3, 4


class ckpt_aor_options(ctypes.Structure):
    _fields_ = [("struct_size", _u32), ("grad_dtype", _u32), ("chunk_bytes", _u64), ("n_slots", _u32),
                ("threads", _u32), ("priority", _i32), ("flags", _u32), ("key", _u64), ("reserved", _u32 * 4)]


class ckpt_aor_shard(ctypes.Structure):
    _fields_ = [("master", _vp), ("grad", _vp), ("bounds", ctypes.POINTER(_u64)), ("m", _u32), ("my_index", _u32)]


class ckpt_aor_stats(ctypes.Structure):
    _fields_ = [(n, _u64) for n in ("steps", "chunks", "d2h_bytes", "h2d_bytes")] + \
               [(n, ctypes.c_double) for n in ("update_s", "stall_s", "last_step_ms")]


class CkptError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        self.code = code
        super().__init__(f"{where}: {ckpt_strerror(code)} ({code}): {msg}")


_lib = None


def lib():
    """The loaded libreft_ckpt.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "ckpt_options_default": (None, [ctypes.POINTER(ckpt_options)]),
            "ckpt_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ckpt_options), ctypes.POINTER(_vp)]),
            "ckpt_destroy": (ctypes.c_int, [_vp]),
            "ckpt_register": (ctypes.c_int, [_vp, ctypes.POINTER(ckpt_tensor), _u64, ctypes.POINTER(ckpt_layout)]),
            "ckpt_geometry": (ctypes.c_int, [_vp, ctypes.POINTER(_u64), ctypes.POINTER(_u64), ctypes.POINTER(_u64),
                                             ctypes.POINTER(_u32)]),
            "ckpt_tensor_offset": (ctypes.c_int, [_vp, _u64, ctypes.POINTER(_u64)]),
            "ckpt_export_handle": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(_u64)]),
            "ckpt_protect": (ctypes.c_int, [_vp, ctypes.POINTER(ckpt_group)]),
            "ckpt_snapshot": (ctypes.c_int, [_vp, _u64, _vp, ctypes.POINTER(_u64)]),
            "ckpt_fence": (ctypes.c_int, [_vp, _u64, _vp]),
            "ckpt_wait": (ctypes.c_int, [_vp, _u64]),
            "ckpt_test": (ctypes.c_int, [_vp, _u64, ctypes.POINTER(ctypes.c_int)]),
            "ckpt_load": (ctypes.c_int, [_vp, _vp]),
            "ckpt_rebuild": (ctypes.c_int, [_vp, _i32, _vp]),
            "ckpt_recover": (ctypes.c_int, [_vp, _u32, _vp]),
            "ckpt_sync": (ctypes.c_int, [_vp]),
            "ckpt_window": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
            "ckpt_has_apply": (ctypes.c_int, [_vp, _u64]),
            "ckpt_has_apply_layers": (ctypes.c_int, [_vp, _u64, _u64]),
            "ckpt_has_plan3": (ctypes.c_int, [_u32, _u32, ctypes.c_double, _u64, ctypes.c_double, ctypes.c_double,
                                              ctypes.POINTER(ckpt_has_plan3_t)]),
            "ckpt_has_plan": (ctypes.c_int, [_u32, _u32, ctypes.c_double, _u64, ctypes.c_double,
                                             ctypes.POINTER(ckpt_has_plan_t)]),
            "ckpt_forget": (ctypes.c_int, [_vp, ctypes.c_uint8]),
            "ckpt_host_view": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_u64),
                                              ctypes.POINTER(_vp), ctypes.POINTER(_u64)]),
            "ckpt_get_stats": (ctypes.c_int, [_vp, ctypes.POINTER(ckpt_stats)]),
            "ckpt_stats_reset": (ctypes.c_int, [_vp]),
            "ckpt_strerror": (ctypes.c_char_p, [ctypes.c_int]),
            "ckpt_last_error": (ctypes.c_char_p, []),
            "ckpt_plan_layout": (ctypes.c_int, [_vp, _u64, _u32, _vp, ctypes.POINTER(_u64)]),
            "ckpt_plan_common": (ctypes.c_int, [_vp, _u32, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
            "ckpt_version": (ctypes.c_char_p, []),
            "ckpt_arena_unlink": (ctypes.c_int, [_u64, _u32, _u32]),
            "ckpt_probe_fabric": (ctypes.c_int, [_vp, ctypes.c_int, _u64, _u32, _vp, ctypes.POINTER(ctypes.c_double)]),
            # include/ckpt_aor.h
            "ckpt_aor_options_default": (None, [ctypes.POINTER(ckpt_aor_options)]),
            "ckpt_aor_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ckpt_aor_options),
                                               ctypes.POINTER(ckpt_aor_shard), ctypes.POINTER(_vp)]),
            "ckpt_aor_destroy": (ctypes.c_int, [_vp]),
            "ckpt_aor_seed": (ctypes.c_int, [_vp, _u64, _vp]),
            "ckpt_aor_step": (ctypes.c_int, [_vp, ctypes.c_float, _vp, ctypes.POINTER(_u64)]),
            "ckpt_aor_fence": (ctypes.c_int, [_vp, _u64, _vp]),
            "ckpt_aor_wait": (ctypes.c_int, [_vp, _u64]),
            "ckpt_aor_restore": (ctypes.c_int, [_vp, _vp, ctypes.POINTER(_u64)]),
            "ckpt_aor_forget": (ctypes.c_int, [_vp, ctypes.c_uint8]),
            "ckpt_aor_view": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_u64), ctypes.POINTER(_u64),
                                             ctypes.POINTER(_u32)]),
            "ckpt_aor_get_stats": (ctypes.c_int, [_vp, ctypes.POINTER(ckpt_aor_stats)]),
            "ckpt_aor_unlink": (ctypes.c_int, [_u64, _u32]),
            "ckpt_aor_apply": (ctypes.c_int, [_vp, _vp, _u32, _u64, ctypes.c_float]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, where: str) -> int:
    if rc < 0:
        raise CkptError(rc, where, ckpt_last_error())
    return rc


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------- messages ---------
def ckpt_strerror(code: int) -> str:
    return lib().ckpt_strerror(code).decode()


def ckpt_last_error() -> str:
    return lib().ckpt_last_error().decode(errors="replace")


def ckpt_version() -> str:
    return lib().ckpt_version().decode()


# ---------------------------------------------------------------- lifecycle --------
def ckpt_options_default(**kw) -> ckpt_options:
    o = ckpt_options()
    lib().ckpt_options_default(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def ckpt_create(device: int, options: Optional[ckpt_options] = None) -> int:
    ctx = _vp()
    _check(lib().ckpt_create(device, ctypes.byref(options) if options is not None else None, ctypes.byref(ctx)),
           "ckpt_create")
    return ctx.value


def ckpt_destroy(ctx: int) -> None:
    _check(lib().ckpt_destroy(ctx), "ckpt_destroy")


_DTYPES = {"bfloat16": CKPT_DTYPE_BF16, "float16": CKPT_DTYPE_FP16, "float32": CKPT_DTYPE_FP32}


def tensor_desc(t, role: int = CKPT_ROLE_OTHER, flags: int = 0, name: str = "") -> tuple:
    """(ptr, nbytes, dtype, role, flags, name) of a torch tensor (must be contiguous)."""
    if not t.is_contiguous():
        raise ValueError("registered tensors must be contiguous")
    return (t.data_ptr(), t.numel() * t.element_size(), _DTYPES.get(str(t.dtype).split(".")[-1], CKPT_DTYPE_BYTES),
            role, flags, name)


def ckpt_register(ctx: int, tensors: Sequence, layout: Optional[dict] = None) -> None:
    """tensors: torch tensors or (ptr, nbytes, dtype, role, flags, name) tuples."""
    arr = (ckpt_tensor * len(tensors))()
    names = []
    for i, t in enumerate(tensors):
        d = t if isinstance(t, tuple) else tensor_desc(t)
        names.append(d[5].encode() if d[5] else None)
        arr[i] = ckpt_tensor(d[0], d[1], d[2], d[3], d[4], 0, names[-1])
    lay = ckpt_layout(**(layout or {}))
    _check(lib().ckpt_register(ctx, arr, len(tensors), ctypes.byref(lay)), "ckpt_register")


def ckpt_geometry(ctx: int) -> dict:
    a, b, c, m = _u64(), _u64(), _u64(), _u32()
    _check(lib().ckpt_geometry(ctx, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(m)),
           "ckpt_geometry")
    return {"L": a.value, "L_star": b.value, "unit": c.value, "m": m.value}


def ckpt_tensor_offset(ctx: int, t: int) -> int:
    o = _u64()
    _check(lib().ckpt_tensor_offset(ctx, t, ctypes.byref(o)), "ckpt_tensor_offset")
    return o.value


def ckpt_export_handle(ctx: int) -> bytes:
    buf = ctypes.create_string_buffer(CKPT_HANDLE_BYTES)
    n = _u64(CKPT_HANDLE_BYTES)
    _check(lib().ckpt_export_handle(ctx, buf, ctypes.byref(n)), "ckpt_export_handle")
    return buf.raw[: n.value]


def ckpt_protect(ctx: int, m: int, my_index: int, transport: int = CKPT_GROUP_IPC,
                 handles: Optional[bytes] = None, members: Optional[Sequence[int]] = None,
                 scheme: int = CKPT_SCHEME_DEFAULT) -> int:
    """Returns CKPT_OK, or CKPT_EUNAVAIL for m == 1 (snapshot-only; not an error)."""
    g = ckpt_group(m, my_index, transport, scheme, None, None)
    keep = None
    if handles is not None:
        keep = ctypes.create_string_buffer(handles, len(handles))
        g.handles = ctypes.cast(keep, _vp)
    if members is not None:
        keep_m = (_vp * len(members))(*members)
        g.members = ctypes.cast(keep_m, ctypes.POINTER(_vp))
    rc = lib().ckpt_protect(ctx, ctypes.byref(g))
    if rc == CKPT_EUNAVAIL:
        return rc
    return _check(rc, "ckpt_protect")


def ckpt_snapshot(ctx: int, bucket_bytes: int = 0, stream=None) -> int:
    sid = _u64()
    _check(lib().ckpt_snapshot(ctx, bucket_bytes, _stream_handle(stream), ctypes.byref(sid)), "ckpt_snapshot")
    return sid.value


def ckpt_fence(ctx: int, sid: int, stream=None) -> None:
    _check(lib().ckpt_fence(ctx, sid, _stream_handle(stream)), "ckpt_fence")


def ckpt_wait(ctx: int, sid: int) -> None:
    _check(lib().ckpt_wait(ctx, sid), "ckpt_wait")


def ckpt_test(ctx: int, sid: int) -> bool:
    d = ctypes.c_int()
    _check(lib().ckpt_test(ctx, sid, ctypes.byref(d)), "ckpt_test")
    return bool(d.value)


def ckpt_load(ctx: int, stream=None) -> None:
    _check(lib().ckpt_load(ctx, _stream_handle(stream)), "ckpt_load")


def ckpt_rebuild(ctx: int, lost_rank: int, stream=None) -> None:
    _check(lib().ckpt_rebuild(ctx, lost_rank, _stream_handle(stream)), "ckpt_rebuild")


def ckpt_recover(ctx: int, lost_mask: int, stream=None) -> None:
    _check(lib().ckpt_recover(ctx, lost_mask, _stream_handle(stream)), "ckpt_recover")


CKPT_WINDOW_BUBBLE, CKPT_WINDOW_COMPUTE, CKPT_WINDOW_COMM = 0x1, 0x2, 0x4


def ckpt_window(ctx: int, open_, stream=None) -> None:
    """Write the HAS window mask on `stream` (True = both windows, False = closed)."""
    if open_ is True:
        open_ = CKPT_WINDOW_BUBBLE | CKPT_WINDOW_COMPUTE
    elif open_ is False:
        open_ = 0
    _check(lib().ckpt_window(ctx, int(open_), _stream_handle(stream)), "ckpt_window")


def ckpt_has_apply(ctx: int, bubble_bytes: int) -> None:
    _check(lib().ckpt_has_apply(ctx, bubble_bytes), "ckpt_has_apply")


def ckpt_has_apply_layers(ctx: int, bubble_bytes: int, compute_bytes: int) -> None:
    _check(lib().ckpt_has_apply_layers(ctx, bubble_bytes, compute_bytes), "ckpt_has_apply_layers")


def ckpt_has_plan3(stage: int, num_stages: int, c_fb_bp_s: float, snapshot_bytes: int, b_io: float,
                   t_compute_s: float) -> dict:
    """Alg 1 extended to HAS Layers 2 and 3 (host-only; reading Q28)."""
    o = ckpt_has_plan3_t()
    _check(lib().ckpt_has_plan3(stage, num_stages, c_fb_bp_s, snapshot_bytes, b_io, t_compute_s, ctypes.byref(o)),
           "ckpt_has_plan3")
    return {"t_ss": o.t_ss, "t_bubble": o.t_bubble, "t_compute": o.t_compute, "bubble_bytes": o.bubble_bytes,
            "compute_bytes": o.compute_bytes, "comm_bytes": o.comm_bytes}


def ckpt_has_plan(stage: int, num_stages: int, c_fb_bp_s: float, snapshot_bytes: int, b_io: float) -> dict:
    """Alg 1's EstimateSnapshotTime / EstimateBubbleTime / SplitParameter (host-only)."""
    o = ckpt_has_plan_t()
    _check(lib().ckpt_has_plan(stage, num_stages, c_fb_bp_s, snapshot_bytes, b_io, ctypes.byref(o)),
           "ckpt_has_plan")
    return {"t_ss": o.t_ss, "t_bubble": o.t_bubble, "bubble_bytes": o.bubble_bytes,
            "compute_bytes": o.compute_bytes}


def ckpt_sync(ctx: int) -> None:
    _check(lib().ckpt_sync(ctx), "ckpt_sync")


def ckpt_probe_fabric(ctx: int, mode: int, bytes_per_peer: int, ctas: int = 0, stream=None) -> float:
    """All-concurrent NVLink pull GB/s of this member (every member must call it at once)."""
    g = ctypes.c_double()
    _check(lib().ckpt_probe_fabric(ctx, mode, bytes_per_peer, ctas, _stream_handle(stream), ctypes.byref(g)),
           "ckpt_probe_fabric")
    return g.value


def ckpt_forget(ctx: int, poison: int = 0xA5) -> None:
    _check(lib().ckpt_forget(ctx, poison), "ckpt_forget")


def ckpt_host_view(ctx: int, which: int = 0, copy: bool = False):
    """(data, parity) numpy uint8 arrays over the completed (0) / ongoing (1) host image.
    Zero-copy views by default: they dangle after ckpt_destroy (pass copy=True to keep)."""
    d, dl, p, pl = _vp(), _u64(), _vp(), _u64()
    _check(lib().ckpt_host_view(ctx, which, ctypes.byref(d), ctypes.byref(dl), ctypes.byref(p), ctypes.byref(pl)),
           "ckpt_host_view")
    data = np.ctypeslib.as_array(ctypes.cast(d.value, ctypes.POINTER(ctypes.c_uint8)), shape=(dl.value,)) \
        if dl.value else np.zeros(0, np.uint8)
    par = np.ctypeslib.as_array(ctypes.cast(p.value, ctypes.POINTER(ctypes.c_uint8)), shape=(pl.value,)) \
        if pl.value else None
    if copy:
        data = data.copy()
        par = par.copy() if par is not None else None
    return data, par


def ckpt_get_stats(ctx: int) -> dict:
    s = ckpt_stats()
    _check(lib().ckpt_get_stats(ctx, ctypes.byref(s)), "ckpt_get_stats")
    return s.as_dict()


def ckpt_stats_reset(ctx: int) -> None:
    _check(lib().ckpt_stats_reset(ctx), "ckpt_stats_reset")


def ckpt_arena_unlink(key: int, m: int, nbuf: int = 2) -> None:
    _check(lib().ckpt_arena_unlink(key, m, nbuf), "ckpt_arena_unlink")


def ckpt_plan_layout(nbytes: Sequence[int], align: int = 256):
    nb = np.ascontiguousarray(np.asarray(nbytes, dtype=np.uint64))
    off = np.zeros(max(len(nb), 1), dtype=np.uint64)
    L = _u64()
    _check(lib().ckpt_plan_layout(nb.ctypes.data, len(nb), align, off.ctypes.data, ctypes.byref(L)),
           "ckpt_plan_layout")
    return off[: len(nb)].astype(np.int64).tolist(), L.value


def ckpt_plan_common(Ls: Sequence[int], unit: int):
    a = np.ascontiguousarray(np.asarray(Ls, dtype=np.uint64))
    Ls_, ue = _u64(), _u64()
    _check(lib().ckpt_plan_common(a.ctypes.data, len(a), unit, ctypes.byref(Ls_), ctypes.byref(ue)),
           "ckpt_plan_common")
    return Ls_.value, ue.value


# ---------------------------------------------------------------- group plumbing ---
def exchange_handles(blob: bytes, group=None) -> bytes:
    """All-gather this rank's fixed-size handle blob over torch.distributed (NCCL or gloo);
    returns the concatenation in group-rank order.  Handshake only."""
    import torch
    import torch.distributed as dist
    assert len(blob) == CKPT_HANDLE_BYTES
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    mine = torch.from_numpy(np.frombuffer(blob, dtype=np.uint8).copy()).to(dev)
    world = dist.get_world_size(group)
    outs = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(outs, mine, group=group)
    return b"".join(bytes(o.cpu().numpy().tobytes()) for o in outs)


def protect_ipc(ctx: int, group=None, scheme: int = CKPT_SCHEME_DEFAULT) -> int:
    """Collective: bind the torch.distributed group (one process per GPU of one node) as
    the protection group; member index = rank in ``group``."""
    import torch.distributed as dist
    blobs = exchange_handles(ckpt_export_handle(ctx), group)
    m, me = dist.get_world_size(group), dist.get_rank(group)
    rc = ckpt_protect(ctx, m, me, CKPT_GROUP_IPC, handles=blobs, scheme=scheme)
    dist.barrier(group)
    return rc


def protect_local(ctxs: Sequence[int], scheme: int = CKPT_SCHEME_DEFAULT) -> None:
    """Bind m contexts of this process (same or different devices) as one group."""
    for i, c in enumerate(ctxs):
        ckpt_protect(c, len(ctxs), i, CKPT_GROUP_LOCAL, members=list(ctxs), scheme=scheme)


# ---------------------------------------------------------------- harness generator
_synth = None


def reft_synth_fill(ptr: int, nbytes: int, seed: int, rank: int, tensor: int, xor_mode: int = 0,
                    stream=None) -> None:
    """Seeded GPU fill (harness generator, include/reft_synth.h)."""
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise ImportError(f"{SYNTH_PATH} is missing: build first")
        _synth = ctypes.CDLL(SYNTH_PATH)
        _synth.reft_synth_fill.restype = ctypes.c_int
        _synth.reft_synth_fill.argtypes = [_vp, _u64, _u64, _u64, _u64, ctypes.c_int, _vp]
    rc = _synth.reft_synth_fill(ptr, nbytes, seed, rank, tensor, xor_mode, _stream_handle(stream))
    if rc != 0:
        raise RuntimeError(f"reft_synth_fill failed ({rc})")


# ---------------------------------------------------------------- AOR (include/ckpt_aor.h) ----
def ckpt_aor_options_default(**kw) -> ckpt_aor_options:
    o = ckpt_aor_options()
    lib().ckpt_aor_options_default(ctypes.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def ckpt_aor_create(device: int, options: ckpt_aor_options, master, grad, bounds: Sequence[int],
                    my_index: int) -> int:
    """master: this member's fp32 optimizer shard (device tensor or pointer); grad: the complete
    flat gradient (device tensor or pointer); bounds: m+1 element offsets of the partition."""
    b = (_u64 * len(bounds))(*[int(x) for x in bounds])
    sh = ckpt_aor_shard(_ptr(master), _ptr(grad), ctypes.cast(b, ctypes.POINTER(_u64)), len(bounds) - 1, my_index)
    a = _vp()
    _check(lib().ckpt_aor_create(device, ctypes.byref(options), ctypes.byref(sh), ctypes.byref(a)), "ckpt_aor_create")
    return a.value


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return x.data_ptr() if x.numel() else 0


def ckpt_aor_destroy(a: int) -> None:
    _check(lib().ckpt_aor_destroy(a), "ckpt_aor_destroy")


def ckpt_aor_seed(a: int, step: int = 0, stream=None) -> None:
    _check(lib().ckpt_aor_seed(a, step, _stream_handle(stream)), "ckpt_aor_seed")


def ckpt_aor_step(a: int, eta: float, stream=None) -> int:
    t = _u64()
    _check(lib().ckpt_aor_step(a, eta, _stream_handle(stream), ctypes.byref(t)), "ckpt_aor_step")
    return t.value


def ckpt_aor_fence(a: int, step: int, stream=None) -> None:
    _check(lib().ckpt_aor_fence(a, step, _stream_handle(stream)), "ckpt_aor_fence")


def ckpt_aor_wait(a: int, step: int) -> None:
    _check(lib().ckpt_aor_wait(a, step), "ckpt_aor_wait")


def ckpt_aor_restore(a: int, stream=None) -> int:
    t = _u64()
    _check(lib().ckpt_aor_restore(a, _stream_handle(stream), ctypes.byref(t)), "ckpt_aor_restore")
    return t.value


def ckpt_aor_forget(a: int, poison: int = 0xA5) -> None:
    _check(lib().ckpt_aor_forget(a, poison), "ckpt_aor_forget")


def ckpt_aor_view(a: int, copy: bool = True):
    """(replica float32 array, step, state) of the replica this member holds."""
    p, n, t, st = _vp(), _u64(), _u64(), _u32()
    _check(lib().ckpt_aor_view(a, ctypes.byref(p), ctypes.byref(n), ctypes.byref(t), ctypes.byref(st)),
           "ckpt_aor_view")
    if n.value == 0:
        arr = np.zeros(0, np.float32)
    else:
        arr = np.ctypeslib.as_array((ctypes.c_float * n.value).from_address(p.value))
        if copy:
            arr = arr.copy()
    return arr, t.value, st.value


def ckpt_aor_get_stats(a: int) -> dict:
    s = ckpt_aor_stats()
    _check(lib().ckpt_aor_get_stats(a, ctypes.byref(s)), "ckpt_aor_get_stats")
    return {n: getattr(s, n) for n, _ in s._fields_}


def ckpt_aor_unlink(key: int, m: int) -> None:
    _check(lib().ckpt_aor_unlink(key, m), "ckpt_aor_unlink")


def ckpt_aor_apply(w: np.ndarray, grad: np.ndarray, eta: float) -> None:
    """Host-only: one Eq 4 step in place on float32 ``w`` (grad float32, or uint16 bf16 bits)."""
    assert w.dtype == np.float32 and w.flags.c_contiguous and grad.flags.c_contiguous and grad.size == w.size
    dt = CKPT_DTYPE_BF16 if grad.dtype == np.uint16 else CKPT_DTYPE_FP32
    assert grad.dtype in (np.uint16, np.float32)
    _check(lib().ckpt_aor_apply(w.ctypes.data, grad.ctypes.data, dt, w.size, eta), "ckpt_aor_apply")


def aor_group_key(group=None) -> int:
    """A random non-zero key chosen by rank 0 of ``group`` and broadcast (torch.distributed)."""
    import torch
    import torch.distributed as dist
    key = int.from_bytes(os.urandom(8), "little") | 1
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor([key & 0x7FFFFFFFFFFFFFFF], dtype=torch.int64, device=dev)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        key = int(t.item())
    return key


def aor_recover(a: int, lost_mask: int, my_index: int, m: int, barrier, stream=None) -> int:
    """The recovery protocol of include/ckpt_aor.h over a group barrier (e.g. dist.barrier):
    survivors drain, lost members restore their master shard from their holder, and the
    owners of the replicas the lost members held re-seed them.  Every member calls this with
    the same lost_mask; returns the step of the restored state (-1 on members that restored
    nothing and seeded nothing)."""
    lost = [(lost_mask >> j) & 1 for j in range(m)]
    if any(lost[j] and lost[(j - 1) % m] for j in range(m)) or (m == 1 and lost[0]):
        raise CkptError(CKPT_EUNRECOVERABLE, "aor_recover", "a lost member's holder is lost too")
    step = -1
    if not lost[my_index]:
        _, step, _ = ckpt_aor_view(a, copy=False)    # drains this member's pending updates
    barrier()
    if lost[my_index]:
        step = ckpt_aor_restore(a, stream)
    barrier()
    if lost[(my_index - 1) % m] and not lost[my_index]:
        ckpt_aor_seed(a, step, stream)   # this member's master is at the group's step
    barrier()
    return step
