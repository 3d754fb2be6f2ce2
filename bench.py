#!/usr/bin/env python
"""Benchmark of the TideGS working-set step (a1-a5) on B200.

One step = tgs_activate(camera batch t) + tgs_step_adam over R n K, i.e. the
whole hot path: cull, residency selection, delta, slot allocation/eviction,
gather of S+ from the pinned host tier, write-back of dirty S-, masked Adam.
Prints ONE JSON line (rank 0).  See DESIGN.md §6 for every field.

  python bench.py [--gpus N --steps K --warmup W] [--config 300m] [--moments cold]
  python bench.py --impl reference ...      # the CPU oracle as the reference arm
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload as W  # noqa: E402

METRIC = "active Gaussians materialised+updated/sec"
ROW_BYTES_ADAM = 1652  # read g, m, v, theta (4 x 236 B) + write theta, m, v (3 x 236 B)
# cold restart (R6): a block's first update after admission reads no m, v (the
# moments are zero): 708 B per active row (read g, theta; write theta) plus its
# whole m, v record written (472 B per row of the block)
ROW_BYTES_ADAM_FRESH = 708
ROW_BYTES_MV = 472


def adam_bytes(rows, fresh_rows, fresh_blocks, B):
    """Algorithmic HBM bytes of k_adam over `rows` active rows, of which
    `fresh_rows` belong to the `fresh_blocks` first-updated (cold-restarted) blocks."""
    return ((rows - fresh_rows) * ROW_BYTES_ADAM + fresh_rows * ROW_BYTES_ADAM_FRESH
            + fresh_blocks * B * ROW_BYTES_MV)


def lr_3dgs():
    lr = np.empty(59, np.float32)
    lr[0:3], lr[3:6], lr[6:51], lr[51], lr[52:55], lr[55:59] = 1.6e-4, 2.5e-3, 1.25e-4, 5e-2, 5e-3, 1e-3
    return lr


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="300m", choices=sorted(W.CONFIGS))
    ap.add_argument("--moments", default="cold", choices=["cold", "persist"])
    ap.add_argument("--start", type=int, default=0, help="first batch index of the trajectory")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    ap.add_argument("--shard-of", type=int, default=0,
                    help="one process measures rank 0's shard of a G-way block-sharded table "
                         "(per-GPU share of a G-GPU run, no collectives; e.g. --config 1b --shard-of 8)")
    ap.add_argument("--no-tide", action="store_true",
                    help="ablation w/o Tide (PAPER.md:570-573): restage R_{t+1} every batch")
    ap.add_argument("--no-overlap", action="store_true",
                    help="ablation w/o Overlap (PAPER.md:576-579): I/O and compute serialised")
    ap.add_argument("--refresh-bounds", action="store_true",
                    help="NEXT f2: conservative bound refresh after every update (R25)")
    ap.add_argument("--fine-filter", action="store_true",
                    help="NEXT f1: Level-2 filter -> I_t mask -> masked Adam in every step")
    ap.add_argument("--store", default=None, metavar="DIR",
                    help="NEXT f3: the shard lives in a log-structured store under DIR (SSD) "
                         "below a CPU cache of --cache-blocks records (PAPER.md:224-251)")
    ap.add_argument("--cache-blocks", type=int, default=0,
                    help="CPU-cache records for --store (0 -> 3x the GPU capacity)")
    ap.add_argument("--store-buffered", action="store_true",
                    help="--store through the page cache instead of O_DIRECT")
    ap.add_argument("--capacity", type=int, default=0,
                    help="override the config's capacity C (blocks, world size 1; C_g = ceil(C/G))")
    ap.add_argument("--pool-slots", type=int, default=0,
                    help="device slot pool P per GPU (0 -> 2 C_g, R13)")
    ap.add_argument("--sync-activate", action="store_true",
                    help="tgs_activate (plan readback every step) instead of tgs_activate_async")
    ap.add_argument("--xfer", default="auto", choices=["auto", "kernel", "ce"],
                    help="a4 transfers: TMA bulk-copy kernels (k_xfer) or copy-engine runs "
                         "(TGS_XFER_COPY_ENGINE, plan readback); auto -> ce, except 11m (in-memory, "
                         "latency-bound: the async activate needs the kernels)")
    ap.add_argument("--no-persist-detail", action="store_true",
                    help="skip the 100m persist measurement the default run adds (detail.persist)")
    ap.add_argument("--prefetch", type=int, default=-1, metavar="BLOCKS",
                    help="--store read-ahead buffers (tgs_prefetch of the next batch every step; "
                         "-1 -> C, 0 -> off)")
    ap.add_argument("--io-threads", type=int, default=0,
                    help="parallel SSD requests of the --store tier (0 -> library default)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.rows = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def link_peak(torch, dev):
    """Measured pinned host<->device copy bandwidth (GB/s) on this box, 1 GiB."""
    n = 1 << 30
    x = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    best = {"h2d": 0.0, "d2h": 0.0}
    for _ in range(3):
        for k, f in (("h2d", lambda: d.copy_(x, non_blocking=True)),
                     ("d2h", lambda: x.copy_(d, non_blocking=True))):
            torch.cuda.synchronize()
            t = time.perf_counter()
            f()
            torch.cuda.synchronize()
            best[k] = max(best[k], n / (time.perf_counter() - t) / 1e9)
    # both directions at once (two streams, 1 GiB each): the ceiling of a step
    # that gathers and writes back concurrently
    y = torch.empty(n, dtype=torch.uint8).pin_memory()
    e = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    best["bidir_h2d"] = best["bidir_d2h"] = 0.0
    for _ in range(3):
        a0, a1, b1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        a0.record()
        s1.wait_event(a0)
        s2.wait_event(a0)
        with torch.cuda.stream(s1):
            d.copy_(x, non_blocking=True)
            a1.record(s1)
        with torch.cuda.stream(s2):
            y.copy_(e, non_blocking=True)
            b1.record(s2)
        torch.cuda.synchronize()
        best["bidir_h2d"] = max(best["bidir_h2d"], n / (a0.elapsed_time(a1) * 1e6))
        best["bidir_d2h"] = max(best["bidir_d2h"], n / (a0.elapsed_time(b1) * 1e6))
    del x, d, y, e
    return best


def ssd_read_peak(path, gib=4):
    """Measured sequential O_DIRECT read bandwidth (GB/s) of the store's disk:
    dd of the first GiBs of the base segment in 16 MiB requests."""
    try:
        out = subprocess.run(["dd", f"if={path}", "of=/dev/null", "bs=16M", f"count={64 * gib}",
                              "iflag=direct"], capture_output=True, text=True, timeout=120).stderr
        line = [x for x in out.splitlines() if "copied" in x][-1]
        nbytes = float(line.split()[0])
        secs = float(line.split(",")[-2].split()[0])
        return nbytes / secs / 1e9
    except Exception:
        return None


def _churn(st0, st1, steps):
    """SURVEY §8d churn over the timed steps (this rank): evictions, dirty
    evictions and re-admissions per step, the share of block updates that
    cold-restarted their moments, and the mean length of a finished residency."""
    d = {k: st1[k] - st0[k] for k in st1}
    return {"evict_per_step": d["n_evict"] / steps,
            "evict_dirty_per_step": d["n_evict_dirty"] / steps,
            "readmissions_per_step": d["readmissions"] / steps,
            "cold_restart_ratio": (d["cold_restart_updates"] / d["total_updates"]
                                   if d["total_updates"] else None),
            "mean_resident_streak": (d["resident_streak_sum"] / d["streak_count"]
                                     if d["streak_count"] else None)}


def _workload(args):
    """The named config, with --capacity overriding its C (the capacity sweep of
    SURVEY §8d: C as a multiple of the mean #K_t)."""
    wl = W.CONFIGS[args.config]
    if args.capacity:
        import dataclasses
        wl = dataclasses.replace(wl, capacity=int(args.capacity))
    return wl


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        # TGS_BENCH_BACKEND=gloo: functional run of the multi-rank path with
        # several ranks sharing one GPU (NCCL refuses duplicate GPUs)
        backend = os.environ.get("TGS_BENCH_BACKEND") or ("nccl" if args.impl == "ours" else "gloo")
        dist.init_process_group(backend)
    return ws, rank, local


def run_reference(args, ws, rank):
    """Reference arm = the CPU oracle as it stands, on the host cores, same
    config / metric; each step a bounded sample of the workload."""
    if rank != 0:
        return
    import oracle as O
    wl = _workload(args)
    sc = wl.scene()
    tr = wl.trajectory(sc)
    if wl.tsp:  # f4 on the reference arm: the oracle's clustered-TSP order
        tr.reorder(O.order_views(tr.features(150.0 if wl.traj == "aerial" else 20.0))[0])
    moments = O.COLD_RESTART if args.moments == "cold" else O.PERSIST
    o = O.Oracle(O.make_config(sc.N, sc.B, wl.capacity, moments=moments), sc.bounds(),
                 fill=None, track_all=True)
    syn = _synth_struct(sc)
    gfn = C.cast(W.lib().wl_grad_cb, C.c_void_p).value
    lr = lr_3dgs()
    times, rows = [], []
    total = args.warmup + args.steps
    budget = 150.0  # seconds of oracle work for the whole run
    t_all = time.perf_counter()
    timed = 0
    for i in range(total):
        t0 = time.perf_counter()
        before = o.stats()["n_active_rows"]
        o.activate(tr.batch_planes(args.start + i, wl.J))
        o.step_adam(lr, grad=(gfn, C.addressof(syn)))
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            rows.append(o.stats()["n_active_rows"] - before)
            timed += 1
        if time.perf_counter() - t_all > budget and timed >= 1:
            break
    o.close()
    value = sum(rows) / sum(times)
    cores = 1
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Gaussians/s",
            "n_gpus": 0, "steps": len(times), "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config_dict(args, wl, ws),
            "cpu_baseline": {"value": value, "unit": "Gaussians/s", "cores": cores,
                             "host": _host_cpu(),
                             "kind": "oracle",
                             "sample": f"oracle (single-thread C++17) from batch {args.start}, "
                                       f"{len(times)} timed of {total} requested steps "
                                       f"(capped at {budget:.0f}s), rows zero-filled"},
            "e2e": {"value": value, "unit": "Gaussians/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _synth_struct(sc):
    class Synth(C.Structure):
        _fields_ = [("seed", C.c_uint64), ("n_gaussians", C.c_uint64),
                    ("block_size", C.c_uint32), ("p32", C.c_uint32)]
    return Synth(W.SEEDS["grads"], sc.N, sc.B, 0)


def _config_dict(args, wl, ws):
    if getattr(args, "shard_of", 0) > 1 and ws == 1:
        d = _config_dict_base(args, wl, args.shard_of)
        d["shard"] = f"rank 0 of a {args.shard_of}-way block-sharded table, measured alone"
        d["world_size"] = 1
        return d
    return _config_dict_base(args, wl, ws)


def _config_dict_base(args, wl, ws):
    order = ("shuffled, then clustered-TSP order (f4)" if wl.tsp else
             "random" if wl.shuffled else "smooth")
    return {"workload": f"{wl.name}: {wl.n_gaussians:,} Gaussians, {wl.traj} trajectory "
                        f"({order} order), J={wl.J} cameras/batch",
            "n_gaussians": wl.n_gaussians, "block_size": wl.block_size, "J": wl.J,
            "capacity_blocks_per_gpu": -(-wl.capacity // ws), "moments": args.moments,
            **({"pool_slots_per_gpu": args.pool_slots} if getattr(args, "pool_slots", 0) else {}),
            "policy": "restage-all (w/o Tide)" if getattr(args, "no_tide", False) else "tide",
            "activate": ("tgs_activate (plan readback)" if (getattr(args, "sync_activate", False)
                         or getattr(args, "store", None) or getattr(args, "no_tide", False)
                         or getattr(args, "pool_slots", 0) or xfer_mode(args) == 1)
                         else "tgs_activate_async"),
            "xfer": ("TMA bulk-copy kernels (k_xfer; store tier)" if getattr(args, "store", None)
                     else "gather: copy-engine runs of consecutive records + k_commit; "
                          "write-back: TMA kernel (k_xfer, 2 CTAs)"
                     if xfer_mode(args) == 1 else "TMA bulk-copy kernels (k_xfer)"),
            "overlap": not getattr(args, "no_overlap", False),
            "bound_refresh": bool(getattr(args, "refresh_bounds", False)),
            "world_size": ws,
            "I_t": "Level-2 fine filter (f1)" if getattr(args, "fine_filter", False) else "all rows of R n K (mask NULL)",
            "l2": "inputs larger than L2 (Adam touches GBs per step)",
            "grads": "synthetic counter-hash gradients resident in the grad pool (renderer out of scope)",
            "host_tier": ("pinned host copy of the shard" if not getattr(args, "store", None) else
                          f"NEXT f3 store: CPU cache of {args.cache_blocks} block records over "
                          f"{'buffered' if args.store_buffered else 'O_DIRECT'} log-structured "
                          "segments (base + patches) on local disk"),
            "seeds": W.SEEDS}


def _gpu_local_core(local):
    """One core of the NUMA node local to GPU `local` (sysfs local_cpulist of its PCI
    device), else the last core of this process's affinity set."""
    allowed = sorted(os.sched_getaffinity(0))
    try:
        import torch
        pr = torch.cuda.get_device_properties(local)
        bdf = "%04x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
        spec = open(f"/sys/bus/pci/devices/{bdf}/local_cpulist").read().strip()
        cores = []
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cores += range(int(lo), int(hi or lo) + 1)
        cores = [c for c in cores if c in allowed]
        if cores:
            return cores[-1]
    except Exception:
        pass
    return allowed[-1]


def cpu_baseline(args, wl, sc, tr, budget_s, shard_ws=1, shard_rank=0, local=0):
    """The oracle as it stands (single thread, pinned to one core on the GPU's
    NUMA node) on a bounded sample of the same workload: it is first advanced
    metadata-only through the batches before the GPU's timed window, then times
    whole steps from the window's first batch on (rows zero-filled), with its
    per-phase clocks (cull / plan / copies / Adam).  --shard-of G: rank 0's shard."""
    import oracle as O
    moments = O.COLD_RESTART if args.moments == "cold" else O.PERSIST
    cap = -(-wl.capacity // shard_ws)
    o = O.Oracle(O.make_config(sc.N, sc.B, cap, moments=moments, world_size=shard_ws,
                               rank=shard_rank), sc.bounds(), fill=None, track_all=False)
    syn = _synth_struct(sc)
    gfn = C.cast(W.lib().wl_grad_cb, C.c_void_p).value
    lr = lr_3dgs()
    first = args.start + args.warmup
    for i in range(args.start, first):  # state of the GPU's timed window, untimed
        o.activate(tr.batch_planes(i, wl.J))
        o.step_adam(lr, grad=(gfn, C.addressof(syn)))
    o.track_all_from_now()
    core = _gpu_local_core(local)
    mask0 = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {core})
    try:
        ph0 = o.phase_seconds()
        t0 = time.perf_counter()
        n = rows = 0
        while True:
            before = o.stats()["n_active_rows"]
            o.activate(tr.batch_planes(first + n, wl.J))
            o.step_adam(lr, grad=(gfn, C.addressof(syn)))
            rows += o.stats()["n_active_rows"] - before
            n += 1
            if time.perf_counter() - t0 > budget_s or n >= 64:
                break
        dt = time.perf_counter() - t0
        ph1 = o.phase_seconds()
    finally:
        os.sched_setaffinity(0, mask0)
    o.close()
    return {"value": rows / dt, "unit": "Gaussians/s", "cores": 1, "kind": "oracle",
            "sample": f"batches {first}..{first + n - 1} (the GPU's timed window onwards), "
                      f"{dt:.1f}s single-thread pinned to core {core}, after a metadata-only "
                      f"pass over batches {args.start}..{first - 1}; rows zero-filled"
                      + (f"; rank 0 of a {shard_ws}-way sharded table" if shard_ws > 1 else ""),
            "phases_s_per_step": {k: (ph1[k] - ph0[k]) / n for k in ph1},
            "host": _host_cpu()}


def _host_cpu():
    """CPU model and logical core count of the box the oracle ran on."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def self_launch(args):
    """`bench.py --gpus N` (N > 1) outside torchrun: re-run this command as N
    ranks of one node through torch.distributed.run (127.0.0.1 rendezvous).
    Rank 0 prints the JSON line; the exit code is the launcher's."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    ws, rank, local = dist_init(args)
    if ws != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; measuring {ws} rank(s)",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import torch
    if os.environ.get("TGS_BENCH_BACKEND") == "gloo":
        local = 0  # every rank on cuda:0 (functional multi-rank run on one GPU)
    torch.cuda.set_device(local)
    line = measure(args, ws, rank, local)
    if persist_detail_wanted(args, ws):
        # the north-star persist policy (moments gathered and scattered with theta)
        # on the largest config whose persist host tier fits this box: 100m
        import copy
        a2 = copy.copy(args)
        a2.config, a2.moments, a2.no_cpu_baseline, a2.capacity = "100m", "persist", True, 0
        l2 = measure(a2, ws, rank, local)
        if rank == 0:
            line["detail"]["persist"] = {
                k: l2[k] for k in ("value", "unit", "ms_per_step", "config", "e2e", "roofline",
                                   "link_roofline", "gpu_launches", "clocks")}
            line["detail"]["persist"]["detail"] = {
                k: l2["detail"][k] for k in ("active_blocks_per_step", "stage_in_blocks_per_step",
                                             "h2d_GB_per_step", "d2h_GB_per_step", "churn",
                                             "locality", "step_ms")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def xfer_mode(args):
    """tgs_xfer of the run: 1 = copy-engine runs (needs the plan readback), 0 = TMA kernels"""
    if getattr(args, "store", None):
        return 0
    if getattr(args, "xfer", "auto") == "auto":
        # copy-engine runs win wherever records move (profiles/ab_xfer_r02.md);
        # 11m in-memory moves none after the fill and is bound by the host's
        # per-step latency, which only the async activate (kernels) removes
        return 0 if args.config == "11m" else 1
    return 1 if args.xfer == "ce" else 0


def persist_detail_wanted(args, ws):
    """the default invocation (300m cold, N = 1) also measures 100m persist"""
    return (ws == 1 and args.config == "300m" and args.moments == "cold" and not args.shard_of
            and not args.store and not args.capacity and not args.no_persist_detail
            and not (args.no_tide or args.no_overlap or args.fine_filter or args.refresh_bounds))


def measure(args, ws, rank, local):
    """One table of args.config through the timed window; rank 0 gets the JSON
    line (dict), the other ranks None.  Frees the table before returning."""
    import torch
    import paper_2605_20150_b200 as P  # noqa: F401
    from paper_2605_20150_b200 import tidegs as T

    dev = torch.device("cuda", local)
    line = None
    wl = _workload(args)
    sc = wl.scene()
    tr = wl.trajectory(sc)
    order_ms = None
    if wl.tsp:  # f4: clustered-TSP order of the (shuffled) views, on the GPU
        focus = 150.0 if wl.traj == "aerial" else 20.0
        perm, _, _, _, order_ms = T.order_views(tr.features(focus), local)
        tr.reorder(perm)
    shard_ws, shard_rank = (args.shard_of, 0) if args.shard_of > 1 and ws == 1 else (ws, rank)
    cap = -(-wl.capacity // shard_ws)
    moments = T.COLD_RESTART if args.moments == "cold" else T.PERSIST
    t_setup = time.perf_counter()
    cfg = T.make_config(sc.N, sc.B, cap, pool_slots=args.pool_slots, moments=moments, world_size=shard_ws, rank=shard_rank,
                        device=local, tide=0 if args.no_tide else 1,
                        serialize=1 if args.no_overlap else 0,
                        refresh_bounds=1 if args.refresh_bounds else 0,
                        level2=1 if args.fine_filter else 0, xfer=xfer_mode(args))
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)  # collectives and timing events on the compute stream
    build_ms = None
    store = None
    if args.store:
        if not args.cache_blocks:
            args.cache_blocks = 3 * cap
        store = dict(dir=os.path.join(args.store, f"rank{shard_rank:03d}"),
                     cache_blocks=args.cache_blocks, direct_io=0 if args.store_buffered else 1,
                     io_threads=args.io_threads,
                     prefetch_blocks=cap if args.prefetch < 0 else args.prefetch)
        os.makedirs(args.store, exist_ok=True)
    if wl.build:  # f2b: Morton-sort + block the unsorted scene on the GPU
        perm, bounds, build_ms = T.build_layout(sc.table_cs(), sc.B, local)
        table = T.Table(cfg, bounds, fill=sc.perm_fill(perm), stream=stream.cuda_stream,
                        store=store)
    else:
        table = T.Table(cfg, sc.bounds(), fill=sc.fill_fn, stream=stream.cuda_stream,
                        store=store)
    setup_s = time.perf_counter() - t_setup
    if ws > 1:  # C1 active-set all-gather / C2 count all-reduce, issued by the library
        table.set_comm(T.torch_comm())
    # synthetic gradients for every slot, written once (renderer out of scope)
    P_ = table.P
    ids = torch.arange(P_, dtype=torch.int32, device=dev) % max(1, table.num_local_blocks)
    ids = ids * shard_ws + shard_rank
    slots = torch.arange(P_, dtype=torch.int32, device=dev)
    act0 = table.activate(np.zeros((0, 6, 4), np.float32))
    W.cuda_lib().wl_cuda_synth_grads(act0.d_grads, act0.grad_stride, ids.data_ptr(),
                                     slots.data_ptr(), P_, sc.B, sc.N, W.SEEDS["grads"], 0,
                                     stream.cuda_stream)
    torch.cuda.synchronize()
    lr = lr_3dgs()
    J = wl.J
    total = args.warmup + args.steps
    planes = [tr.batch_planes(args.start + i, J) for i in range(total)]

    fmask = torch.zeros((table.P, (sc.B + 31) // 32), dtype=torch.int32, device=dev) \
        if args.fine_filter else None

    steplog = os.environ.get("TGS_BENCH_STEPLOG")  # per-step Adam counters (ncu runs only:
    steplog = open(steplog, "w") if steplog else None  # each line syncs the device)

    def step(i, cams=None):
        _step(i, cams)
        if steplog:
            t, st = table.timing(), table.stats()
            steplog.write(json.dumps({"step": i, "rows": st["n_active_rows"],
                                      "fresh_rows": t["fresh_active_rows"],
                                      "fresh_blocks": t["fresh_blocks"],
                                      "active_blocks": st["n_active_blocks"], "B": sc.B}) + "\n")
            steplog.flush()

    use_async = not (args.sync_activate or args.store or args.no_tide or args.pool_slots
                     or xfer_mode(args) == 1)

    def _step(i, cams=None):
        pl = planes[i] if cams is None else cams
        act = table.activate_async(pl) if use_async else table.activate(pl)
        if fmask is not None:
            table.fine_filter(fmask.data_ptr())
        table.step_adam(lr, mask_ptr=fmask.data_ptr() if fmask is not None else None)
        if store and store["prefetch_blocks"] and i + 2 < total:
            table.prefetch(planes[i + 2], 2)  # f3 read-ahead, two batches ahead

    for i in range(args.warmup):
        step(i)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    table.set_profiling(True)
    st0 = table.stats()
    tm0 = table.timing()
    ss0 = table.store_stats() if store else None
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # e2e over the same timed steps: each step's camera batch comes from pinned
    # host memory and its result (the step's counters) goes back to pinned host
    # memory (tgs_get_stats_async); the wall clock stops when every read landed
    e2e_on = not args.no_e2e
    nf = len(T.STAT_FIELDS)
    if e2e_on:
        res = torch.zeros((args.steps + 1, nf), dtype=torch.int64).pin_memory()
        host_planes = [torch.from_numpy(planes[i].copy()).pin_memory()
                       for i in range(args.warmup, total)]
        table.stats_async(res[0].data_ptr())
        torch.cuda.synchronize()
    with Clocks(local) as clk:
        t_wall0 = time.perf_counter()
        ev0.record(stream)
        # per-step cadence on the compute stream (no host sync): p50 / p99 of T_iter
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for j, i in enumerate(range(args.warmup, total)):
            if e2e_on:
                step(i, host_planes[j].numpy())
                table.stats_async(res[j + 1].data_ptr())
            else:
                step(i)
            evs[j].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    step_ms = np.diff(np.array([0.0] + [ev0.elapsed_time(e) for e in evs]))
    if ws > 1:
        torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1)
    st1 = table.stats()
    store_detail = None
    if store:
        ss1 = table.store_stats()
        dd = {k: ss1[k] - ss0[k] for k in ss1 if k not in ("cached", "cached_dirty")}
        store_detail = {"per_step": {k: v / args.steps for k, v in dd.items()},
                        "hit_rate": dd["hits"] / max(1, dd["hits"] + dd["misses"]),
                        "ssd_read_GBps_in_reads": (dd["read_bytes"] / (dd["read_ms"] / 1e3) / 1e9
                                                   if dd["read_ms"] else None),
                        "ssd_write_GBps_in_appends": (dd["write_bytes"] / (dd["write_ms"] / 1e3)
                                                      / 1e9 if dd["write_ms"] else None),
                        "cached": ss1["cached"], "cached_dirty": ss1["cached_dirty"]}
    tm = table.timing()
    rows = st1["n_active_rows"] - st0["n_active_rows"]
    rows_local = rows
    fresh_rows = tm["fresh_active_rows"] - tm0["fresh_active_rows"]
    fresh_blocks = tm["fresh_blocks"] - tm0["fresh_blocks"]
    h2d = st1["h2d_bytes"] - st0["h2d_bytes"]
    d2h = st1["d2h_bytes"] - st0["d2h_bytes"]
    stage_in = st1["n_stage_in"] - st0["n_stage_in"]
    visible = st1["n_visible"] - st0["n_visible"]
    active_blocks = st1["n_active_blocks"] - st0["n_active_blocks"]
    # this rank's host-link bytes of the timed steps: S+ records gathered over
    # PCIe (not those re-admitted from the write-back ring in HBM) and dirty S-
    rec_b = sc.B * 59 * 4 * (3 if args.moments == "persist" else 1)
    ring_recs = tm["h2d_ring_records"] - tm0["h2d_ring_records"]
    # PCIe bytes: the transfer kernels skip ring re-admissions (read from HBM); the
    # copy engines move whole runs, re-admitted records included (k_commit then
    # takes the ring copy)
    ce = xfer_mode(args) == 1
    h2d_link, d2h_link = (h2d if ce else h2d - ring_recs * rec_b), d2h
    if ws > 1:  # whole job: counts summed over ranks, the slowest rank's clock
        t = torch.tensor([rows, ms, h2d, d2h, stage_in, visible, tm["adam_ms"], active_blocks],
                         dtype=torch.float64, device=dev)
        mx = t.clone()
        torch.distributed.all_reduce(t)
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        rows, h2d, d2h, stage_in, visible, active_blocks = (
            float(x) for x in (t[0], t[2], t[3], t[4], t[5], t[7]))
        ms = float(mx[1])
    value = rows / (ms / 1e3)

    # ---- e2e: the same metric through the public API from host buffers: every
    #      step copies its camera batch from pinned host memory (activate) and
    #      reads its result (the step's counters) back to pinned host memory
    #      (tgs_get_stats_async); the clock stops when every read has landed.
    e2e = None
    if e2e_on:
        n_e = args.steps
        dt, dev_s = t_wall, ev0.elapsed_time(ev1) / 1e3
        fi = {n: j for j, n in enumerate(T.STAT_FIELDS)}
        d_rows = int(res[n_e, fi["n_active_rows"]] - res[0, fi["n_active_rows"]])
        d_h2d = int(res[n_e, fi["h2d_bytes"]] - res[0, fi["h2d_bytes"]])
        d_d2h = int(res[n_e, fi["d2h_bytes"]] - res[0, fi["d2h_bytes"]])
        if ws > 1:  # whole job: rows and bytes summed over ranks, the slowest rank's clock
            import torch.distributed as dist
            tsum = torch.tensor([d_rows, d_h2d, d_d2h], dtype=torch.float64, device=dev)
            tmax = torch.tensor([dt, dev_s], dtype=torch.float64, device=dev)
            dist.all_reduce(tsum)
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            d_rows, d_h2d, d_d2h = (int(x) for x in tsum.tolist())
            dt, dev_s = tmax.tolist()
        e2e = {"value": d_rows / dt, "unit": "Gaussians/s",
               "h2d_bytes_per_step": int((d_h2d + n_e * J * 96) / n_e),
               "d2h_bytes_per_step": int((d_d2h + n_e * nf * 8) / n_e),
               "ms_per_step": 1e3 * dt / n_e,
               "device_value_same_steps": d_rows / dev_s,
               "how": "wall clock over the %d timed steps (the device-timed window): pinned "
                      "host planes in, per-step async stats readback to pinned host memory, "
                      "one sync at the end" % n_e}

    hbm_peak, peak_kind = peaks()
    # this rank's k_adam launches: its rows, its fresh rows, its launch time
    adam_ms = tm["adam_ms"] / max(1, tm["adam_launches"])
    adam_bpl = adam_bytes(rows_local, fresh_rows, fresh_blocks, sc.B) / max(1, args.steps)
    achieved = adam_bpl / (adam_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_adam_r02.json")
    if os.path.exists(tp):  # ncu --set full capture of a k_adam launch of this workload
        tj = json.load(open(tp))
        traffic = {"dram_bytes_per_launch": tj["traffic_bytes"],
                   "algorithmic_bytes_same_launch": tj["algorithmic_bytes"],
                   "ratio": tj["traffic_over_algorithmic"], "source": tj["source"]}
    roof = {"bound": "hbm", "kernel": "k_adam", "achieved": achieved, "peak": hbm_peak,
            "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
            "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": adam_bpl,
            "algorithmic_bytes_rule": "1652 B per active row; first update of a cold-restarted "
                                      "block: 708 B per active row + 472 B per row of the block "
                                      "(m, v record written, not read)",
            "fresh_row_share": fresh_rows / max(1, rows_local),
            "avg_launch_ms": adam_ms,
            "note": ("k_adam is the dominant device-memory kernel; the host link "
                     "(link_roofline: copy-engine run copies, or the k_xfer TMA kernels) "
                     "bounds the step when records move")}
    lp = link_peak(torch, dev) if rank == 0 else None
    if store and store_detail is not None:
        store_detail["ssd_read_peak_GBps"] = ssd_read_peak(os.path.join(store["dir"], "base.tdgs"))
    link = None
    if rank == 0:
        h2d_rate = h2d_link / (tm["h2d_ms"] / 1e3) / 1e9 if tm["h2d_ms"] else None
        d2h_rate = d2h_link / (tm["d2h_ms"] / 1e3) / 1e9 if tm["d2h_ms"] else None
        link = {"bound": "host-link", "h2d_achieved": h2d_rate, "d2h_achieved": d2h_rate,
                "h2d_peak": lp["h2d"], "d2h_peak": lp["d2h"], "unit": "GB/s",
                "h2d_frac": (h2d_rate / lp["h2d"]) if h2d_rate else None,
                "d2h_frac": (d2h_rate / lp["d2h"]) if d2h_rate else None,
                "bidir_h2d_peak": lp["bidir_h2d"], "bidir_d2h_peak": lp["bidir_d2h"],
                "bidir_h2d_frac": (h2d_rate / lp["bidir_h2d"]) if h2d_rate else None,
                "bidir_d2h_frac": (d2h_rate / lp["bidir_d2h"]) if d2h_rate else None,
                "peak_kind": "measured in this run: pinned 1 GiB cudaMemcpy, one direction "
                             "alone (h2d/d2h_peak) and both at once on two streams (bidir_*)",
                "how": ("h2d: copy-engine spans (CUDA events around each step's run copies "
                        "on the h2d stream); d2h: the write-back kernel's spans (k_xfer, 2 CTAs, "
                        "d2h stream); each over the bytes it moved" if ce else
                        "k_xfer gather / write-back kernel spans (CUDA events on the h2d / d2h "
                        "streams) over the records they moved across PCIe"),
                "ring_readmissions_per_step": ring_recs / args.steps,
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, wl, sc, tr, args.cpu_sample_s, shard_ws, shard_rank, local)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "Gaussians/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": _config_dict(args, wl, ws),
                "clocks": clk.summary(), "e2e": e2e, "gpu_launches": tm["kernel_launches"],
                "roofline": roof, "link_roofline": link, "cpu_baseline": cpu,
                "detail": {"active_blocks_per_step": None if not args.steps else
                           active_blocks / args.steps,
                           "visible_blocks_per_step": visible / args.steps,
                           "stage_in_blocks_per_step": stage_in / args.steps,
                           "h2d_GB_per_step": h2d / args.steps / 1e9,
                           "d2h_GB_per_step": d2h / args.steps / 1e9,
                           "churn": _churn(st0, st1, args.steps),
                           "locality": {
                               "mean_K_over_Kloc": (st1["n_visible"] - st0["n_visible"])
                               / args.steps / max(1, table.num_local_blocks),
                               "jaccard_consecutive_K": (
                                   (st1["k_inter_sum"] - st0["k_inter_sum"])
                                   / max(1, st1["k_union_sum"] - st0["k_union_sum"])),
                               "stage_in_over_visible": (st1["n_stage_in"] - st0["n_stage_in"])
                               / max(1, st1["n_visible"] - st0["n_visible"]),
                               "how": "rank 0 over the timed steps: mean |K_t| / K_loc (paper "
                                      "~3.5%, PAPER.md:139), the consecutive-batch Jaccard "
                                      "sum |K_t n K_t+1| / sum |K_t u K_t+1|, and sum |S+| / "
                                      "sum |K_t|: the Tide / w/o-Tide traffic ratio (paper "
                                      "0.10 / 0.85 GB = 0.12, PAPER.md:522, 572)"},
                           "step_ms": {"p50": float(np.percentile(step_ms, 50)),
                                       "p99": float(np.percentile(step_ms, 99)),
                                       "max": float(step_ms.max()),
                                       "how": "compute-stream event after each step (rank 0)"},
                           "plan_ms_per_step": tm["plan_ms"] / args.steps,
                           "fine_ms_per_step": tm["fine_ms"] / args.steps,
                           "adam_prologue_ms_per_step": tm["adam_prologue_ms"] / args.steps,
                           "evict_pack_ms_per_step": tm["evict_ms"] / args.steps,
                           "h2d_ms_per_step": tm["h2d_ms"] / args.steps,
                           "d2h_ms_per_step": tm["d2h_ms"] / args.steps,
                           "setup_s": setup_s, "layout_build_gpu_ms": build_ms,
                           "view_order_gpu_ms": order_ms,
                           "store": store_detail}}
    table.close()
    del table
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if store and os.environ.get("TGS_KEEP_STORE") != "1":
        import shutil
        shutil.rmtree(store["dir"], ignore_errors=True)
    return line


if __name__ == "__main__":
    main()
