#!/usr/bin/env python3
"""Pinned D2H bandwidth by host-buffer kind, all ranks at once (torchrun):
cudaHostAlloc (torch pin_memory) vs anonymous mmap (+/- THP) + cudaHostRegister,
one 4 GiB copy vs 4 x 1 GiB copies."""
import ctypes
import json
import mmap
import os

import torch
import torch.distributed as dist

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(rank)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
N = 4 << 30
db = torch.empty(N, dtype=torch.uint8, device="cuda")
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
libc = ctypes.CDLL("libc.so.6")
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]


def host_registered(thp):
    p = libc.mmap(None, N, 3, 0x22 | 0x4000, -1, 0)  # PROT_RW, MAP_PRIVATE|ANON|NORESERVE
    if thp:
        libc.madvise(p, N, 14)  # MADV_HUGEPAGE
    ctypes.memset(p, 0, N)
    r = torch.cuda.cudart().cudaHostRegister(p, N, 1)
    assert int(r) == 0, r
    arr = (ctypes.c_uint8 * N).from_address(p)
    return torch.frombuffer(arr, dtype=torch.uint8)


def timed(h, chunks):
    best = 0
    for _ in range(3):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step = N // chunks
        for i in range(chunks):
            h[i * step:(i + 1) * step].copy_(db[i * step:(i + 1) * step], non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, N / e0.elapsed_time(e1) / 1e6)
    return round(best, 2)


res = {}
hp = torch.empty(N, dtype=torch.uint8, pin_memory=True)
res["cudaHostAlloc_1x4G"] = timed(hp, 1)
res["cudaHostAlloc_4x1G"] = timed(hp, 4)
del hp
hr = host_registered(True)
res["mmap_thp_reg_1x4G"] = timed(hr, 1)
res["mmap_thp_reg_4x1G"] = timed(hr, 4)
res["mmap_thp_reg_16x256M"] = timed(hr, 16)
hn = host_registered(False)
res["mmap_4k_reg_1x4G"] = timed(hn, 1)
if rank == 0:
    print(json.dumps(res))
if world > 1:
    dist.destroy_process_group()
