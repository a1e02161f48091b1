"""Box probe: host RAM/cores/topology, pinned D2H/H2D GB/s with
1..N GPUs concurrent, P2P copy GB/s between GPU pairs. Plain torch; harness only."""
import os, sys, time, json, subprocess, threading
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["free_g"] = sh("free -g")
out["nproc"] = sh("nproc").strip()
out["lscpu"] = sh("lscpu | head -30")
out["topo"] = sh("nvidia-smi topo -m")
out["numa"] = sh("ls /sys/devices/system/node/ | grep node")
out["smi"] = sh("nvidia-smi --query-gpu=index,name,pci.bus_id,clocks.sm,clocks.max.sm --format=csv")
ng = torch.cuda.device_count()
out["ngpu"] = ng
NB = 1 << 30

def d2h_bw(dev, nbytes, direction, res, key, reps=5):
    torch.cuda.set_device(dev)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    t0 = time.time()
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    res[key + "_pin_s"] = time.time() - t0
    s = torch.cuda.Stream(dev)
    best = 0
    with torch.cuda.stream(s):
        for i in range(reps + 1):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if direction == "d2h":
                h.copy_(d, non_blocking=True)
            else:
                d.copy_(h, non_blocking=True)
            e1.record(s)
            e1.synchronize()
            if i:
                best = max(best, nbytes / e0.elapsed_time(e1) / 1e6)
    res[key] = best

for direction in ("d2h", "h2d"):
    for n in [1, 2, 4, 8]:
        if n > ng:
            break
        res = {}
        ths = [threading.Thread(target=d2h_bw, args=(i, NB, direction, res, f"g{i}")) for i in range(n)]
        [t.start() for t in ths]; [t.join() for t in ths]
        out[f"{direction}_conc{n}"] = res
        print(direction, n, res, flush=True)

# P2P
if ng >= 2:
    p2p = {}
    for a in range(ng):
        for b in range(ng):
            if a == b: continue
            ok = torch.cuda.can_device_access_peer(a, b)
            x = torch.empty(NB // 4, dtype=torch.uint8, device=a)
            y = torch.empty(NB // 4, dtype=torch.uint8, device=b)
            torch.cuda.synchronize(a)
            for i in range(3):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                with torch.cuda.device(b):
                    e0.record(); y.copy_(x); e1.record(); e1.synchronize()
            p2p[f"{a}->{b}"] = (ok, (NB // 4) / e0.elapsed_time(e1) / 1e6)
    out["p2p_copy_gbs"] = p2p
    print(p2p)
# stream memop support via driver attribute
try:
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    err, dev = cu.cuDeviceGet(0)
    for name in ["CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR_V2", "CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS_V2"]:
        a = getattr(cu.CUdevice_attribute, name, None)
        if a is not None:
            out[name] = cu.cuDeviceGetAttribute(a, dev)[1]
except Exception as e:
    out["memop_probe_err"] = repr(e)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k not in ("lscpu", "topo")}, indent=1))
print(out["topo"]); print(out["lscpu"])
