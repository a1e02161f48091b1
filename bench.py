#!/usr/bin/env python3
"""bench.py -- REFT snapshot-and-protect on B200 (driver contract).

One step = one full snapshot+protect of the rank's registered state: gather-pack
kernel -> (N >= 2: rotated XOR parity over NVLink P2P) -> copy-engine D2H into the
ongoing pinned host image -> commit on every rank (ckpt_snapshot + ckpt_wait).

  python bench.py [--gpus N --steps K --warmup W] [--config c2_7b_tp8] [--impl reference]

N = 1 runs snapshot only (a group of one has no redundancy); N >= 2 is launched under
torchrun, one process per GPU, and the N ranks form one protection group (m = N).
value = state bytes committed per GPU per second (GB/s per GPU, weak scaling); the
aggregate over all N GPUs is `aggregate_gbs`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "snapshot+parity GB/s per GPU at 1/2/4/8 B200; co-running GEMM slowdown %"
NVLINK_PEAK_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction (nominal 900)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=8)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2_7b_tp8")
    p.add_argument("--bucket", type=int, default=512 << 20)
    p.add_argument("--n-slots", type=int, default=0, help="0 = full device copy (single-launch pack)")
    p.add_argument("--unit", type=int, default=1 << 20, help="stripe unit u (Q4; 1 MiB: DESIGN 11b)")
    p.add_argument("--pack", default="tma", choices=["lsu", "tma", "ce"],
                   help="pack kernel: 128-bit LSU, TMA bulk through SMEM, or copy engines (zero SMs)")
    p.add_argument("--gather", default="kernel", choices=["kernel", "ce"],
                   help="parity: XOR kernel reads peers over NVLink, or copy engines pull units first")
    p.add_argument("--encode", default="pull", choices=["pull", "push"],
                   help="parity encode: pull (row owner reads its peers' units over NVLink) or push (every "
                        "member XOR-reduces its units into the row owners' parity, CKPT_OPT_XOR_PUSH)")
    p.add_argument("--device-only", action="store_true",
                   help="CKPT_OPT_DEVICE_ONLY: device-side protect only (pack + parity into HBM, no D2H)")
    p.add_argument("--max-ctas", type=int, default=0, help="CTA budget of a pack/XOR launch (0 = 2 x SMs)")
    p.add_argument("--group-size", type=int, default=0,
                   help="protection group size m (0 = all N ranks); N/m disjoint node subgroups")
    p.add_argument("--scheme", default="aec", choices=["aec", "arc", "arc_aec"],
                   help="protection: AEC parity (default), ARC ring copies, or both (collaborative)")
    p.add_argument("--no-corun", action="store_true", help="skip the co-running GEMM measurement")
    p.add_argument("--corun-pairs", type=int, default=12, help="A/B window pairs of the co-run measurement")
    p.add_argument("--no-paper-shape", action="store_true",
                   help="N=1: skip the extra short measurement of C4 (Llama-2-34B TP8, the paper's workload shape)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    return p.parse_args()


def trace(*a):
    if os.environ.get("BENCH_TRACE"):
        print(f"[rank {os.environ.get('RANK', 0)} {time.strftime('%H:%M:%S')}]", *a, file=sys.stderr, flush=True)


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ clocks ----------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(gpu)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait(10)
        rows = [r.split(", ") for r in open(self.f.name).read().strip().splitlines() if r.count(",") >= 8]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


class NvmlSampler:
    """SM clock, power and clock-event reasons of one GPU every few ms on a host thread
    (NVML), between start() and stop(): the co-run windows are ~0.4 s, too short for the
    nvidia-smi loop.  stop() -> {"sm_mhz": mean, "power_w": mean, "power_cap": bool}."""

    def __init__(self, torch, dev, period_s: float = 0.005):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            p = torch.cuda.get_device_properties(dev)  # the same GPU whatever CUDA_VISIBLE_DEVICES says
            try:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0")
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(dev.index or 0)
            self.ok = True
        except Exception:
            pass
        self.period = period_s

    def start(self):
        import threading
        self.samples, self.run = [], True
        if not self.ok:
            return

        def loop():
            nv, h = self.nv, self.h
            while self.run:
                try:
                    self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                         nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                         nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                except Exception:
                    pass
                time.sleep(self.period)
        self.t = threading.Thread(target=loop, daemon=True)
        self.t.start()

    def stop(self):
        self.run = False
        if not self.ok:
            return None
        self.t.join()
        if not self.samples:
            return None
        cap = self.nv.nvmlClocksEventReasonSwPowerCap
        return {"sm_mhz": statistics.mean(x[0] for x in self.samples),
                "power_w": statistics.mean(x[1] for x in self.samples),
                "power_cap_frac": sum(1 for x in self.samples if x[2] & cap) / len(self.samples),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU oracle ------
class OracleGroup:
    """The unchanged oracle on `threads` host threads at once for an m-member group: thread i
    takes its own window of stripes of every member's image (windows cut through tensors;
    a stripe-aligned window is exactly what O3/O4/O6 compute for those stripes) and runs
    pack (O3) of every member, the parity of every row (O4) and the rebuild of member 0
    (O6) on it.  Inputs are generated once, before any clock starts; run() times one pass."""

    def __init__(self, config: str, m: int, seconds: float, threads: int, unit: int = 1 << 20):
        import bisect

        import oracle
        import synth

        self.oracle, self.m, self.threads, self.u, self.config = oracle, m, threads, unit, config
        stripe = (m - 1) * self.u if m > 1 else 65536
        specs = [synth.config_tensors(config, j) for j in range(m)]
        nb = [[s_.nbytes for s_ in sp] for sp in specs]
        offs = [oracle.layout(x)[0] for x in nb]
        Lmin = min(oracle.layout(x)[1] for x in nb)
        budget = int(min(max(0.6e9 * seconds * threads, 64 << 20), 4 << 30))  # state bytes, all members
        W = max(stripe, budget // (threads * m) // stripe * stripe)
        self.W = min(W, max(stripe, Lmin // threads // stripe * stripe))

        def pieces(j, a_, b_):
            ps, wh = [], []
            t = max(0, bisect.bisect_right(offs[j], a_) - 1)
            while t < len(nb[j]) and offs[j][t] < b_:
                lo, hi = max(a_, offs[j][t]), min(b_, offs[j][t] + nb[j][t])
                if lo < hi:
                    ps.append(synth.fill(synth.SEED, j, t, hi - offs[j][t])[lo - offs[j][t]:])
                    wh.append(lo - a_)
                t += 1
            return ps, wh

        self.work = [[pieces(j, i * self.W, (i + 1) * self.W) for j in range(m)] for i in range(threads)]
        self.state_bytes = self.W * m * threads
        self.rebuilt_bytes = self.W * threads if m > 1 else 0
        self.desc = (f"oracle pack{' + rotated XOR parity of every row + rebuild of member 0' if m > 1 else ''} of "
                     f"{threads} windows x {self.W / 2**20:.0f} MiB of each of {m} member(s) of {config}, one "
                     f"window per host thread ({threads} threads, each the unchanged 1-thread oracle)")

    def run(self, keep: bool = False) -> float:
        """One timed pass; with keep, self.out[i] = (images, parity rows, rebuilt member 0)
        of window i (the CPU test checks them against the oracle on whole images)."""
        import threading
        o, m, u = self.oracle, self.m, self.u
        self.out = [None] * self.threads

        def one(i):
            Ds = [o.pack(ps, wh, self.W) for ps, wh in self.work[i]]
            Ps = R = None
            if m > 1:
                Ps = [o.encode(Ds, u, r) for r in range(m)]
                R = o.rebuild([None] + Ds[1:], [None] + Ps[1:], u, 0, [True] + [False] * (m - 1))
            if keep:
                self.out[i] = (Ds, Ps, R)

        th = [threading.Thread(target=one, args=(i,)) for i in range(self.threads)]
        t0 = time.perf_counter()
        for x in th:
            x.start()
        for x in th:
            x.join()
        return time.perf_counter() - t0


def oracle_sample(config: str, m: int, seconds: float, step_seed: int = 0, unit: int = 1 << 20):
    """Time the CPU oracle (as it stands) on a bounded sample of the workload: the first
    tensors of each of the m ranks (up to a byte budget sized for ~`seconds` of work),
    pack (O3) and, for m >= 2, the parity of every rank (O4).  Returns (GB/s of state,
    sample description)."""
    import numpy as np

    import oracle
    import synth

    def run(budget):
        imgs, tot = [], 0
        for j in range(m):
            specs = synth.config_tensors(config, j)
            ts, acc = [], 0
            for t, s in enumerate(specs):
                if acc >= budget:
                    break
                n = min(s.nbytes, budget - acc)
                ts.append(synth.fill(synth.SEED + step_seed, j, t, n))
                acc += n
            off, L = oracle.layout([x.size for x in ts])
            imgs.append((ts, off, L))
            tot += acc
        Ls = max(x[2] for x in imgs)
        Lstar, u = oracle.common_length([x[2] for x in imgs], unit) if m > 1 else (Ls, unit)
        t0 = time.perf_counter()
        Ds = [oracle.pack(ts, off, Lstar) for ts, off, _ in imgs]
        if m > 1:
            for r in range(m):
                oracle.encode(Ds, u, r)
        dt = time.perf_counter() - t0
        return tot, dt

    tot, dt = run(32 << 20)
    rate = tot / dt
    budget = int(min(max(rate * seconds / m, 32 << 20), 3 << 30))
    tot, dt = run(budget)
    desc = (f"oracle pack{' + rotated XOR parity of every rank' if m > 1 else ''} of the first "
            f"{budget / 2**20:.0f} MiB of each of {m} rank(s) of {config} (1 thread, gcc -O2)")
    return tot / dt / 1e9, desc, tot, dt


def reference_arm(a, rank, world):
    """The oracle as it stands, on every host core (one window of stripes per thread), for the
    same workload and group size as our arm: one step = pack (O3) of every member + parity
    of every row (O4) + rebuild of member 0 (O6) on a bounded sample (inputs generated once,
    before the clock).  value = state GB/s per member (the group's rate / m), the unit of our
    arm's per-GPU value."""
    if rank != 0:
        return 0
    m = max(world, a.gpus)
    nthr = os.cpu_count() or 1
    og = OracleGroup(a.config, m, max(a.cpu_seconds / max(a.steps, 1), 1.0), nthr, a.unit)
    for _ in range(a.warmup):
        og.run()
    t_all = sum(og.run() for _ in range(a.steps))
    value = og.state_bytes * a.steps / t_all / 1e9 / m
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": m,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(t_all / a.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": a.config, "m": m, "sample": og.desc,
                       "same_config": "same workload and m as our arm; a bounded window of every member per step"},
            "aggregate_gbs": round(value * m, 4),
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": nthr, "kind": "oracle",
                             "sample": og.desc},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm ---------
def main():
    a = parse()
    if os.environ.get("BENCH_WATCHDOG_S"):
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["BENCH_WATCHDOG_S"]), exit=True)
    rank, local, world = env_rank()
    if a.impl == "reference":
        return reference_arm(a, rank, world)
    import torch
    import torch.distributed as dist

    from paper_2310_12670_b200 import build as B
    from paper_2310_12670_b200 import ckpt as C
    from synth.gpu import descriptors, make_rank_state

    if rank == 0 and not os.path.exists(C.LIB_PATH):
        B.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    N = world

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    specs, ts = make_rank_state(a.config, rank, dev)
    trace("state ready")
    S = sum(s.nbytes for s in specs)
    # HOST_LOAD: e2e's ckpt_load must restore from the host image (an H2D per step), never
    # from the still-valid device copy; it does not touch the snapshot path
    flags = (C.CKPT_OPT_TIMING | C.CKPT_OPT_HOST_LOAD | (C.CKPT_OPT_TMA_PACK if a.pack == "tma" else 0)
             | (C.CKPT_OPT_LSU_PACK if a.pack == "lsu" else 0)
             | (C.CKPT_OPT_CE_PACK if a.pack == "ce" else 0) | (C.CKPT_OPT_CE_GATHER if a.gather == "ce" else 0)
             | (C.CKPT_OPT_DEVICE_ONLY if a.device_only else 0) | (C.CKPT_OPT_XOR_PUSH if a.encode == "push" else 0))
    if a.device_only:
        a.n_slots = 0
    # pinned host arena per rank and buffer: L + L/(m-1) (AEC) [+ the ARC copy of the
    # neighbour: L (+ L/(m-1))]; fall back to one buffer if the node's available memory
    # (and /dev/shm for the ARC schemes), all ranks together +25%, would not hold two
    scheme = {"aec": C.CKPT_SCHEME_AEC, "arc": C.CKPT_SCHEME_ARC, "arc_aec": C.CKPT_SCHEME_ARC_AEC}[a.scheme]
    Gm = a.group_size or world
    P = S // (Gm - 1) if Gm > 1 and a.scheme != "arc" else 0
    per_buf = S + P + ((S + P) if a.scheme != "aec" and Gm > 1 else 0)
    host_buffers = 2
    try:
        avail = int([l for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0].split()[1]) * 1024
        if a.scheme != "aec":
            st_shm = os.statvfs("/dev/shm")
            avail = min(avail, st_shm.f_bavail * st_shm.f_frsize)
        if world * 2 * per_buf * 1.25 + world * (4 << 30) > avail:  # all ranks of the node
            host_buffers = 1
    except Exception:
        pass
    if a.scheme != "aec":
        flags |= C.CKPT_OPT_SHM_ARENA
    opts = C.ckpt_options_default(n_slots=a.n_slots, bucket_bytes=a.bucket, stripe_unit=a.unit, flags=flags,
                                  max_ctas=a.max_ctas, host_buffers=host_buffers)
    ctx = C.ckpt_create(local, opts)
    t_setup = time.perf_counter()
    C.ckpt_register(ctx, descriptors(ts, specs), {"rank": rank, "world": world, "local_rank": local,
                                                  "local_world": world, "tp_rank": rank, "tp_size": 8,
                                                  "pp_rank": 0, "pp_size": 1, "dp_rank": 0, "dp_size": 1})
    G = a.group_size or world
    if world % G:
        raise SystemExit(f"--group-size {G} must divide N = {world}")
    sub = None
    if world > 1 and G < world:  # disjoint subgroups of G consecutive ranks
        for s0 in range(0, world, G):
            grp = dist.new_group(list(range(s0, s0 + G)))
            if s0 <= rank < s0 + G:
                sub = grp
    if world > 1 and G > 1:
        C.protect_ipc(ctx, group=sub, scheme=scheme)
    else:
        C.ckpt_protect(ctx, 1, 0)  # EUNAVAIL: snapshot only, allocates the host arena
    t_setup = time.perf_counter() - t_setup
    trace("protected", t_setup)
    g = C.ckpt_geometry(ctx)
    m = g["m"]
    stream = torch.cuda.current_stream()

    # host-link roofline, measured live: D2H of 4 GiB by every rank at once (barrier-
    # aligned) into host memory of the same kind as the arena (THP mmap + cudaHostRegister)
    nprobe = 4 << 30
    hb = registered_host_buffer(torch, nprobe)
    db = torch.empty(nprobe, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(5):  # best of 5: with N >= 2 the ranks' copies share host links, alignment varies
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for o in range(0, nprobe, 512 << 20):  # in 512 MiB copies, like the snapshot's buckets
            hb.t[o:o + (512 << 20)].copy_(db[o:o + (512 << 20)], non_blocking=True)
        e1.record()
        e1.synchronize()
        best = max(best, nprobe / e0.elapsed_time(e1) / 1e6)
    d2h_peak = best
    del db
    hb.release()

    # NVLink roofline, measured live (N >= 2, protected): every member pulls from all of its
    # m-1 peers at once -- the encode's all-to-all pattern -- with the XOR kernel's own bulk
    # load mechanism (SM) and with copy engines (CE); best of 3, barrier-aligned
    fabric = None
    if m >= 2 and scheme != C.CKPT_SCHEME_ARC:
        per_peer = min(1 << 30, (g["L"] // (m - 1)) // 16384 * 16384)
        fabric = {"bytes_per_peer": per_peer}
        for name, mode in (("sm_pull", C.CKPT_PROBE_SM_PULL), ("ce_pull", C.CKPT_PROBE_CE_PULL)):
            vals = []
            for _ in range(3):
                barrier()
                torch.cuda.synchronize()
                vals.append(C.ckpt_probe_fabric(ctx, mode, per_peer, 0, stream))
            fabric[name + "_gbs_rank0"] = round(max(vals), 1)
            fabric[name + "_gbs_min_over_ranks"] = round(-allmax(-max(vals)), 1)
        fabric["note"] = ("ckpt_probe_fabric: all members pull bytes_per_peer from each of their m-1 peers at "
                          "once; sm_pull = cp.async.bulk loads on the XOR kernel's CTA budget (its roofline), "
                          "ce_pull = one copy-engine copy per peer")

    def step():
        sid = C.ckpt_snapshot(ctx, a.bucket, stream)
        C.ckpt_wait(ctx, sid)

    for i in range(a.warmup):
        step()
        trace("warmup step", i)
    C.ckpt_stats_reset(ctx)
    barrier()
    torch.cuda.synchronize()
    p_ = torch.cuda.get_device_properties(dev)  # nvidia-smi -i by PCI bus id: immune to CUDA_VISIBLE_DEVICES
    clk = Clocks(f"{p_.pci_domain_id:08X}:{p_.pci_bus_id:02X}:{p_.pci_device_id:02X}.0")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    t_ms = allmax(e0.elapsed_time(e1))
    st = C.ckpt_get_stats(ctx)
    total_state = allsum(S) * a.steps
    aggregate = total_state / (t_ms / 1e3) / 1e9
    value = aggregate / N  # the metric is GB/s PER GPU (weak scaling: every GPU snapshots its own shard)
    wire = st["d2h_bytes"] / (e0.elapsed_time(e1) / 1e3) / 1e9  # this rank's host-link GB/s

    # dominant kernel roofline (launch durations timed with events on its stream)
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    kern = []
    if st["pack_launches"] and a.pack != "ce":
        per = st["pack_bytes"] / st["pack_launches"]
        dur = st["pack_ms"] / st["pack_launches"]
        kern.append(("pack", st["pack_ms"], {"bound": "hbm", "achieved": per / dur / 1e6, "peak": hbm_peak,
                                             "unit": "GB/s",
                                             "kernel": ("pack_all_kernel" if a.n_slots == 0 else "pack_kernel")
                                             if a.pack == "lsu" else
                                             ("pack_all_tma_kernel" if a.n_slots == 0 else "pack_tma_kernel"),
                                             "bytes_per_launch": per, "avg_launch_us": dur * 1e3,
                                             "launches": st["pack_launches"],
                                             "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy r+w)"}))
    xor_name = ("xor_push_kernel" if a.encode == "push" else
                "xor_kernel<m-1>" if os.environ.get("CKPT_XOR_IMPL") == "lsu" else "xor_tma_kernel<m-1>")
    if st["xor_launches"] and a.gather == "kernel":
        per = st["xor_bytes_in"] / st["xor_launches"]
        dur = st["xor_ms"] / st["xor_launches"]
        live = fabric.get("sm_pull_gbs_min_over_ranks") if fabric else None
        kern.append(("xor", st["xor_ms"], {"bound": "nvlink", "achieved": per / dur / 1e6,
                                           "peak": live or NVLINK_PEAK_GBS,
                                           "unit": "GB/s", "kernel": xor_name, "bytes_per_launch": per,
                                           "avg_launch_us": dur * 1e3, "launches": st["xor_launches"],
                                           "frac_of_770": round(per / dur / 1e6 / NVLINK_PEAK_GBS, 4),
                                           "peak_source": ("live all-concurrent NVLink pull probe (ckpt_probe_fabric "
                                                           "sm_pull, min over ranks), this run" if live else
                                                           "B200_PROFILING.md measured peer copy 770 GB/s/direction")}))
    elif st["xor_launches"]:  # CE gather: the XOR kernel reads local HBM (m-1 streams) and writes parity
        per = (st["xor_bytes_in"] + st["xor_bytes_out"]) / st["xor_launches"]
        dur = st["xor_ms"] / st["xor_launches"]
        kern.append(("xor", st["xor_ms"], {"bound": "hbm", "achieved": per / dur / 1e6, "peak": hbm_peak,
                                           "unit": "GB/s", "kernel": xor_name, "bytes_per_launch": per,
                                           "avg_launch_us": dur * 1e3, "launches": st["xor_launches"],
                                           "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy r+w)"}))
    kern.sort(key=lambda x: -x[1])
    roof = kern[0][2] if kern else None
    if roof:
        roof["frac"] = roof["achieved"] / roof["peak"]
        # per-launch traffic from one ncu capture of this kernel, config AND group size m;
        # for the NVLink-bound XOR it is the NVLink receive user bytes (nvlrx__bytes_data_user),
        # for the HBM-bound pack DRAM read + write; null when no capture exists for this m
        tr_path = os.path.join(ROOT, "profiles", f"traffic_{roof['kernel'].split('<')[0]}_{a.config}_m{m}.json")
        tr = json.load(open(tr_path)) if os.path.exists(tr_path) else {}
        roof["traffic"] = tr.get("bytes_per_launch")
        roof["traffic_metric"] = tr.get("metric")
        roof["traffic_source"] = os.path.relpath(tr_path, ROOT) if tr else None
        for k in ("achieved", "frac", "avg_launch_us"):
            roof[k] = round(roof[k], 4)
    # m = 2 with the copy-engine gather: the parity is a mirror (P.459) pulled by the copy
    # engine straight into the parity buffer -- no kernel, so not a roofline candidate;
    # reported against the live all-concurrent copy-engine pull probe
    ce_mirror = None
    if st.get("gather_ops") and st["gather_ms"] > 0:
        per_step = g["L_star"]
        dur = st["gather_ms"] / max(1, st["snapshots"])
        live = fabric.get("ce_pull_gbs_min_over_ranks") if fabric else None
        ce_mirror = {"bound": "nvlink", "engine": "copy engine (cudaMemcpyAsync peer -> parity), zero SMs",
                     "achieved": round(per_step / dur / 1e6, 2), "peak": live or NVLINK_PEAK_GBS,
                     "unit": "GB/s", "bytes_per_snapshot": per_step, "ms_per_snapshot": round(dur, 3),
                     "copies_per_snapshot": st["gather_ops"] // max(1, st["snapshots"]),
                     "peak_source": "live all-concurrent copy-engine pull probe (ckpt_probe_fabric ce_pull, min over "
                                    "ranks), this run" if live else "B200_PROFILING.md 770 GB/s"}
        ce_mirror["frac"] = round(ce_mirror["achieved"] / ce_mirror["peak"], 4)
    # E9 analog (P.469: erasure coding at 12-15x the snapshot rate): the XOR encode's
    # in-situ NVLink GB/s over this rank's host-link (D2H wire) GB/s
    e9 = None
    xk = [d for k, _, d in kern if k == "xor"] or ([ce_mirror] if ce_mirror else [])
    if xk and wire > 0:
        e9 = {"value": round(xk[0]["achieved"] / wire, 2), "xor_gbs": round(xk[0]["achieved"], 1),
              "d2h_wire_gbs": round(wire, 2), "paper": "12-15x (P.469)"}
    others = {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in d.items()} for k, _, d in kern[1:]}
    launches = int(allsum(st["pack_launches"] + st["xor_launches"]))

    # co-running bf16 GEMM (the O_in-mem analog, P.234; HAS layer 2, P.423)
    # e2e through the public API: load (H2D of the completed image into the tensors)
    # + snapshot + commit (D2H), host wall clock, max over ranks
    e2e = None
    if not a.no_e2e and not a.device_only:
        C.ckpt_stats_reset(ctx)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            C.ckpt_load(ctx, stream)
            step()
        torch.cuda.synchronize()
        barrier()
        te = allmax(time.perf_counter() - t0)
        st2 = C.ckpt_get_stats(ctx)
        e2e = {"value": round(allsum(S) * a.steps / te / 1e9 / N, 4), "unit": "GB/s (per GPU)",
               "h2d_bytes_per_step": int(st2["h2d_bytes"] // a.steps),
               "d2h_bytes_per_step": int(st2["d2h_bytes"] // a.steps),
               "what": "ckpt_load (restore from the completed host image) + ckpt_snapshot + ckpt_wait per step, "
                       "host wall clock, max over ranks"}

    corun = None
    if not a.no_corun:
        corun = {"this_config": gemm_corun(torch, C, ctx, stream, a.bucket, barrier, allmax, dev, a.corun_pairs)}
    C.ckpt_destroy(ctx)  # one context (and one pinned arena) alive at a time
    ctx = None
    if not a.no_corun and a.pack != "ce" and not a.device_only:
        # the zero-SM configuration a training job would use while GEMMs run: copy-engine
        # pack (+ copy-engine gather of the peer units when protected)
        o2 = C.ckpt_options_default(n_slots=a.n_slots, bucket_bytes=a.bucket, stripe_unit=a.unit,
                                    host_buffers=host_buffers,
                                    flags=C.CKPT_OPT_TIMING | C.CKPT_OPT_HOST_LOAD | C.CKPT_OPT_CE_PACK
                                    | (C.CKPT_OPT_CE_GATHER if world > 1 and G > 1 else 0))
        ctx2 = C.ckpt_create(local, o2)
        C.ckpt_register(ctx2, descriptors(ts, specs))
        if world > 1 and G > 1:
            C.protect_ipc(ctx2, group=sub)
        else:
            C.ckpt_protect(ctx2, 1, 0)
        corun["ce_pack"] = gemm_corun(torch, C, ctx2, stream, a.bucket, barrier, allmax, dev, a.corun_pairs)
        C.ckpt_destroy(ctx2)
        # the fine-grained configuration: a ring of 4 small slots (4 MiB buckets, or one
        # stripe when that is larger) with the per-bucket TMA pack -- the C3 sweep at m = 4
        # measured ~0% whole-window slowdown with 4 MiB buckets against 6.5-8% at 512 MiB
        # (profiles/r02/r02l_c3_m4.jsonl); the tensors are released only after the last D2H
        gm = G if world > 1 and G > 1 else 1
        small = max(4 << 20, (gm - 1) * a.unit)
        o3 = C.ckpt_options_default(n_slots=4, bucket_bytes=small, stripe_unit=a.unit, host_buffers=host_buffers,
                                    flags=C.CKPT_OPT_TIMING | C.CKPT_OPT_HOST_LOAD | C.CKPT_OPT_TMA_PACK)
        ctx3 = C.ckpt_create(local, o3)
        C.ckpt_register(ctx3, descriptors(ts, specs))
        if world > 1 and G > 1:
            C.protect_ipc(ctx3, group=sub)
        else:
            C.ckpt_protect(ctx3, 1, 0)
        corun["ring_small_buckets"] = gemm_corun(torch, C, ctx3, stream, small, barrier, allmax, dev, a.corun_pairs)
        corun["ring_small_buckets"]["config"] = {"n_slots": 4, "bucket_bytes": small, "pack": "tma (per bucket)"}
        corun["ring_small_buckets"]["state_gbs_per_gpu_alone"] = round(
            S / (corun["ring_small_buckets"]["snapshot_ms_alone"] / 1e3) / 1e9, 3)
        C.ckpt_destroy(ctx3)
    if corun:  # headline: the configuration whose throughput is the headline (both reported)
        corun["slowdown_pct"] = corun["this_config"]["slowdown_pct"]
        corun["slowdown_pct_config"] = "this_config"

    # N = 1: the paper's own workload shape (C4, Llama-2-34B TP8 stage-0 rank) in the same
    # launch configuration, a few steps -- not the headline (BASELINE's metric is quoted on C2)
    paper_shape = None
    if world == 1 and not a.no_paper_shape and a.config != "c4_34b_tp8_stage0":
        specs4, ts4 = make_rank_state("c4_34b_tp8_stage0", 0, dev)
        S4 = sum(s.nbytes for s in specs4)
        ctx4 = C.ckpt_create(local, C.ckpt_options_default(n_slots=a.n_slots, bucket_bytes=a.bucket, stripe_unit=a.unit,
                                                           host_buffers=host_buffers, max_ctas=a.max_ctas, flags=flags))
        C.ckpt_register(ctx4, descriptors(ts4, specs4))
        C.ckpt_protect(ctx4, 1, 0)
        for _ in range(2):
            sid = C.ckpt_snapshot(ctx4, a.bucket, stream)
            C.ckpt_wait(ctx4, sid)
        C.ckpt_stats_reset(ctx4)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(3):
            sid = C.ckpt_snapshot(ctx4, a.bucket, stream)
            C.ckpt_wait(ctx4, sid)
        f1.record(stream)
        torch.cuda.synchronize()
        t4 = f0.elapsed_time(f1) / 3
        st4 = C.ckpt_get_stats(ctx4)
        paper_shape = {"workload": "c4_34b_tp8_stage0", "state_bytes_per_gpu": S4, "tensors_per_gpu": len(specs4),
                       "steps": 3, "ms_per_step": round(t4, 3), "value": round(S4 / t4 / 1e6, 3), "unit": "GB/s",
                       "host_link_frac": round(st4["d2h_bytes"] / 3 / (t4 / 1e3) / 1e9 / d2h_peak, 4),
                       "pack_gbs": round(st4["pack_bytes"] / st4["pack_ms"] / 1e6, 1) if st4["pack_ms"] else None,
                       "pack_frac_of_hbm": round(st4["pack_bytes"] / st4["pack_ms"] / 1e6 / hbm_peak, 4)
                       if st4["pack_ms"] else None}
        C.ckpt_destroy(ctx4)
        del ts4

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        gbs, desc, _, _ = oracle_sample(a.config, 1, a.cpu_seconds, unit=a.unit)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": desc}
        nthr = os.cpu_count() or 1
        og = OracleGroup(a.config, 1, min(a.cpu_seconds, 8.0), nthr, a.unit)
        dt = og.run()
        cpu["all_cores"] = {"value": round(og.state_bytes / dt / 1e9, 4), "unit": "GB/s", "cores": nthr,
                            "kind": "oracle", "sample": og.desc}
        # the oracle's encode and rebuild (O4, O6) on all cores for a 4-member group: the
        # host-side counterpart of the parity work a protected N >= 2 step does
        og = OracleGroup(a.config, 4, min(a.cpu_seconds, 8.0), nthr, a.unit)
        dt = og.run()
        cpu["parity_all_cores_m4"] = {"value": round(og.state_bytes / dt / 1e9 / 4, 4),
                                      "unit": "GB/s per member", "group_gbs": round(og.state_bytes / dt / 1e9, 4),
                                      "rebuild_gbs": round(og.rebuilt_bytes / dt / 1e9, 4), "cores": nthr,
                                      "kind": "oracle", "sample": og.desc}
        del og

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": N, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(t_ms / a.steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": a.config, "state_bytes_per_gpu": S, "tensors_per_gpu": len(specs),
                       "m": m, "L_star": g["L_star"], "stripe_unit": g["unit"], "bucket_bytes": a.bucket,
                       "n_slots": a.n_slots, "pack": a.pack, "gather": a.gather, "encode": a.encode, "device_only": a.device_only,
                       "max_ctas": a.max_ctas or "2 x SMs", "host_buffers": host_buffers,
                       "scheme": a.scheme, "groups": f"{world // (a.group_size or world)} x m={a.group_size or world}",
                       "l2": f"inputs {S / 1e9:.2f} GB/GPU >> 126 MB L2; no flush needed"},
            "aggregate_gbs": round(aggregate, 3),
            "fabric": fabric,
            "e9_ratio": e9,
            "host_link": None if a.device_only else {
                "achieved_wire_gbs_rank0": round(wire, 3), "peak_d2h_gbs_rank0_measured": round(d2h_peak, 3),
                "frac": round(wire / d2h_peak, 4), "note": "binding roofline of the whole step: pinned D2H of data + parity"},
            "roofline": roof, "other_kernels": others, "ce_mirror": ce_mirror,
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e, "cpu_baseline": cpu, "gemm_corun": corun, "paper_shape": paper_shape,
            "setup_s_rank0": round(t_setup, 2),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


class _Registered:
    """Anonymous THP mmap + cudaHostRegister (the library's arena kind) as a torch tensor."""

    def __init__(self, torch, n):
        import ctypes
        import mmap
        self.m = mmap.mmap(-1, n, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        try:
            self.m.madvise(mmap.MADV_HUGEPAGE)
        except Exception:
            pass
        self.buf = (ctypes.c_uint8 * n).from_buffer(self.m)
        ctypes.memset(self.buf, 0, n)
        self.ptr = ctypes.addressof(self.buf)
        self.cudart = torch.cuda.cudart()
        r = self.cudart.cudaHostRegister(self.ptr, n, 1)
        if int(r) != 0:
            raise RuntimeError(f"cudaHostRegister failed: {r}")
        self.t = torch.frombuffer(self.buf, dtype=torch.uint8)

    def copy_(self, src, non_blocking=True):
        return self.t.copy_(src, non_blocking=non_blocking)

    def release(self):
        self.cudart.cudaHostUnregister(self.ptr)
        del self.t
        del self.buf
        self.m.close()


def registered_host_buffer(torch, n):
    return _Registered(torch, n)


def gemm_corun(torch, C, ctx, stream, bucket, barrier, allmax, dev, pairs=12):
    """bf16 8192^3 GEMMs back to back on a HIGH-priority stream; slowdown while a snapshot
    runs on the library's low-priority streams (the O_in-mem analog, P.234-236; HAS Layer 2,
    P.423).  `pairs` interleaved pairs of windows (alone, with snapshot) in ABBA order, each >= 2x a
    snapshot; the with-snapshot windows also give an in-window slowdown against their own
    GEMMs after the commit.
    Every GEMM is bracketed by its own CUDA events, so besides the whole window the slowdown
    is also reported over the GEMMs that overlap the pack kernel (the pack window) and the
    device-side protect (pack + XOR), located relative to an event recorded on the caller
    stream at the snapshot's capture point.  Times are max over ranks per window."""
    n = 8192
    A = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    Bm = torch.randn(n, n, dtype=torch.bfloat16, device=dev)
    hi = torch.cuda.Stream(device=dev, priority=-5)
    with torch.cuda.stream(hi):
        for _ in range(3):
            torch.matmul(A, Bm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(hi)
    with torch.cuda.stream(hi):
        for _ in range(10):
            torch.matmul(A, Bm)
    e1.record(hi)
    e1.synchronize()
    per = e0.elapsed_time(e1) / 10
    sid = C.ckpt_snapshot(ctx, bucket, stream)
    C.ckpt_wait(ctx, sid)
    snap_ms = C.ckpt_get_stats(ctx)["last_snapshot_ms"] or 250.0
    iters = int(allmax(int(max(20, 2.0 * snap_ms / per))))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]

    nvml = NvmlSampler(torch, dev)

    def window(with_snap):
        barrier()
        torch.cuda.synchronize()
        nvml.start()
        es = torch.cuda.Event(enable_timing=True)
        sid = None
        st0 = C.ckpt_get_stats(ctx)
        es.record(stream)
        if with_snap:
            sid = C.ckpt_snapshot(ctx, bucket, stream)
        with torch.cuda.stream(hi):
            for g0, g1 in ev:
                g0.record(hi)
                torch.matmul(A, Bm)
                g1.record(hi)
        if sid is not None:
            C.ckpt_wait(ctx, sid)
        ev[-1][1].synchronize()
        clk.append(nvml.stop())
        st1 = C.ckpt_get_stats(ctx)
        total = ev[0][0].elapsed_time(ev[-1][1])
        spans = [(es.elapsed_time(g0), es.elapsed_time(g1)) for g0, g1 in ev]
        pack = (st1["pack_ms"] - st0["pack_ms"]) / max(1, st1["pack_launches"] - st0["pack_launches"]) \
            if st1["pack_launches"] > st0["pack_launches"] else 0.0
        xor = (st1["xor_ms"] - st0["xor_ms"]) if st1["xor_launches"] > st0["xor_launches"] else 0.0
        snap = st1["last_snapshot_ms"] if with_snap else None
        return allmax(total), spans, pack, xor, snap

    def overlap_mean(spans, lo, hi_):
        d = [b - a for a, b in spans if b > lo and a < hi_]
        return (sum(d) / len(d), len(d)) if d else (None, 0)

    rows, clk = [], []
    for i in range(pairs):
        # ABBA order: the GEMM slows as the GPU warms up, so alternate which window runs first
        if i % 2 == 0:
            ta, sa, _, _, _ = window(False)
            tw, sw, pack, xor, snap = window(True)
        else:
            tw, sw, pack, xor, snap = window(True)
            ta, sa, _, _, _ = window(False)
        base = sum(b - a for a, b in sa[2:]) / max(1, len(sa) - 2)  # per-GEMM time alone (warm)
        pw, npw = overlap_mean(sw, 0.0, pack)
        dw, ndw = overlap_mean(sw, 0.0, pack + xor)
        sn, nsn = overlap_mean(sw, 0.0, snap or 0.0)
        # in-window baseline: the same window's GEMMs that start after the snapshot committed
        # (same clocks and temperature as the overlapped ones)
        tail = [b - a for a, b in sw if snap and a > snap + 1.0]
        tl = sum(tail) / len(tail) if len(tail) >= 5 else None
        ca, cw = (clk[-2], clk[-1]) if i % 2 == 0 else (clk[-1], clk[-2])
        rows.append({"sm_mhz_alone": ca and round(ca["sm_mhz"], 1), "sm_mhz_with": cw and round(cw["sm_mhz"], 1),
                     "power_w_alone": ca and round(ca["power_w"], 1), "power_w_with": cw and round(cw["power_w"], 1),
                     "power_cap_frac_alone": ca and round(ca["power_cap_frac"], 3),
                     "power_cap_frac_with": cw and round(cw["power_cap_frac"], 3),
                     "clock_drop_pct": (ca["sm_mhz"] / cw["sm_mhz"] - 1) * 100 if ca and cw else None,
                     "whole_pct": (tw / ta - 1) * 100,
                     "in_window_pct": (sn / tl - 1) * 100 if sn and tl else None, "tail_gemms": len(tail),
                     "pack_window_pct": (pw / base - 1) * 100 if pw else None, "pack_window_gemms": npw,
                     "protect_window_pct": (dw / base - 1) * 100 if dw else None,
                     "snapshot_window_pct": (sn / base - 1) * 100 if sn else None,
                     "alone_ms": ta, "with_ms": tw, "pack_ms": pack, "xor_ms": xor, "snapshot_ms": snap})

    def summ(key):
        v = [r[key] for r in rows if r[key] is not None]
        if not v:
            return None
        return {"median": round(statistics.median(v), 3), "min": round(min(v), 3), "max": round(max(v), 3),
                "spread": round(max(v) - min(v), 3)}

    flops = 2 * n ** 3 * iters
    whole = summ("whole_pct")
    return {"slowdown_pct": whole["median"], "whole_window": whole, "in_window": summ("in_window_pct"),
            "clock_drop_pct": summ("clock_drop_pct"),
            "sm_mhz": {"alone": summ("sm_mhz_alone"), "with": summ("sm_mhz_with")},
            "power_w": {"alone": summ("power_w_alone"), "with": summ("power_w_with")},
            "power_cap_frac": {"alone": summ("power_cap_frac_alone"), "with": summ("power_cap_frac_with")},
            "pack_window": summ("pack_window_pct"), "protect_window": summ("protect_window_pct"),
            "snapshot_window": summ("snapshot_window_pct"),
            "pairs": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()} for r in rows],
            "gemm_iters": iters, "gemm_tflops_alone": round(flops / statistics.median([r["alone_ms"] for r in rows]) / 1e9, 1),
            "snapshot_ms_alone": round(snap_ms, 3),
            "window": (f"{pairs} interleaved pairs in ABBA order; whole = GEMM window (>= 2x snapshot, max over ranks); "
                       "in_window = GEMMs overlapping the snapshot vs the same window's GEMMs after its commit; "
                       "pack / protect / snapshot window = mean per-GEMM time of the GEMMs overlapping "
                       "[capture, +pack] / [capture, +pack+xor] / [capture, +snapshot] vs the warm per-GEMM "
                       "time alone (this rank)")}


if __name__ == "__main__":
    sys.exit(main())
