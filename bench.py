"""Benchmark: powersort keys/s on the BASELINE workload (config 2: n=1e7 int32 random runs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C] [--algo powersort]

One JSON line on rank 0.  A "step" is one powersort of one synthetic batch.

ours      value: device-resident throughput; each step restores the unsorted
          input from an HBM copy and flushes L2 (a 512 MiB write) OUTSIDE the
          timed region, then times exactly the sort with CUDA events.
          e2e:   the same sort through the public API `powersort(pinned tensor)`:
          H2D of the keys, sort, D2H of the keys and the Metrics, per step.
          roofline: the executor kernel (leaf formation + every merge), timed
          with CUDA events on its own launch stream; algorithmic bytes
          2*B*(merge_cost + n) per launch.
          cpu_baseline: the C oracle (restatement of the reference powersort)
          on all host cores, one independent copy per thread, bounded sample.
reference the same C oracle port on all host cores (the reference itself is
          pure Python and cannot travel to the GPU box), as its own JSON line.

N > 1 (torchrun): every rank holds a contiguous shard of one global array of
N x n keys; each rank powersorts its shard on its GPU, then a splitter-
partitioned exchange over NCCL and a stable merge give the globally sorted
array (weak scaling, n per GPU).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PEAKS = os.path.join(REPO, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
KERNELS_PER_SORT = 3  # our launches per powersort (see csrc/runsort_b200.cu run_powersort)
ALGO_CODES = {"powersort": 0, "peeksort": 1}  # rs_algo (include/runsort_b200.h)
METRIC = "powersort keys/s at n=1e7 int32 random-runs; % of HBM roofline; 1/2/4/8 GPU"


def hbm_peak():
    try:
        with open(PEAKS) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/rs_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}",
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 7:
                    continue
                try:
                    sm.append(float(f[0]))
                    mx.append(float(f[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except FileNotFoundError:
            pass
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline
def cpu_oracle_throughput(keys: np.ndarray, tags, seconds: float, threads: int, algo: str = "powersort"):
    """Oracle (C restatement of reference powersort / peeksort) on `threads` host
    threads, each sorting its own copies of the workload until ~`seconds` elapse."""
    from oracle import oracle

    oracle.lib()
    sort = getattr(oracle, algo)
    t0 = time.perf_counter()
    a = keys.copy()
    sort(a, 24, "bitonic", None if tags is None else tags.copy())
    single = time.perf_counter() - t0
    reps = max(1, int(seconds / max(single, 1e-3)))

    def work(_):
        for _ in range(reps):
            b = keys.copy()
            sort(b, 24, "bitonic", None if tags is None else tags.copy())
        return reps

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        done = sum(ex.map(work, range(threads)))
    wall = time.perf_counter() - t0
    return done * len(keys) / wall, dict(
        sorts=done, threads=threads, wall_s=round(wall, 3), single_sort_s=round(single, 4))


# ------------------------------------------------------------ workloads
def make_input(cfg: int, n_override=None, seed=1, rank=0):
    from paper_1805_04154_b200 import workloads

    if cfg == 5:
        raise SystemExit("config 5 bench: use --config 5 via bench_multi (device generated)")
    keys, tags = workloads.generate(cfg, n_override, seed + rank)
    return keys, tags


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1805_04154_b200 as rs
    from paper_1805_04154_b200 import _lib

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L = _lib.lib()
    keys_np, tags_np = make_input(args.config, args.n, rank=rank)
    n = len(keys_np)
    kb = keys_np.itemsize
    tb = tags_np.itemsize if tags_np is not None else 0
    B = kb + tb
    src = torch.from_numpy(keys_np).to(dev)
    tsrc = torch.from_numpy(tags_np).to(dev) if tags_np is not None else None
    work = torch.empty_like(src)
    twork = torch.empty_like(tsrc) if tsrc is not None else None
    key_code = _lib.RS_KEY_I32 if kb == 4 else _lib.RS_KEY_I64
    ws_bytes = L.rs_workspace_bytes(ALGO_CODES[args.algo], key_code, tb, n, 24)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    import ctypes

    def one_sort(profile=False, out=None):
        return L.rs_sort(ALGO_CODES[args.algo], key_code, work.data_ptr(), tb, twork.data_ptr() if twork is not None else None,
                         n, 24, 0, ws.data_ptr(), ws_bytes, stream.cuda_stream,
                         ctypes.byref(out) if out is not None else None, None)

    # correctness of the timed path vs the oracle (outside timing)
    work.copy_(src)
    if twork is not None:
        twork.copy_(tsrc)
    m = _lib.RsMetrics()
    _lib.check(one_sort(out=m))
    metrics = dict(merge_cost=int(m.merge_cost), comparisons=int(m.comparisons),
                   runs_detected=int(m.runs_detected), max_stack_height=int(m.max_stack_height))

    L.rs_profile(0)  # the timed steps carry no phase events (kernels launch back to back)
    phase = np.zeros(3)
    exec_elems = None
    for _ in range(args.warmup):
        work.copy_(src)
        if twork is not None:
            twork.copy_(tsrc)
        flush.fill_(1)
        _lib.check(one_sort())
    torch.cuda.synchronize()
    clocks = Clocks(local_rank)
    clocks.start()
    time.sleep(0.3)
    total_ms = 0.0
    exec_ms = []
    buf = (ctypes.c_double * 4)()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        work.copy_(src)
        if twork is not None:
            twork.copy_(tsrc)
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(one_sort())
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    torch.cuda.synchronize()
    clk = clocks.stop()
    # phase split and the merge kernel's own time (roofline): the same steps
    # again with CUDA events between the kernels, outside the timed total
    L.rs_profile(1)
    for _ in range(args.steps):
        work.copy_(src)
        if twork is not None:
            twork.copy_(tsrc)
        flush.fill_(1)
        _lib.check(one_sort())
        torch.cuda.synchronize()
        k = L.rs_profile_read(buf, 4)
        if k >= 3:
            phase += np.array(buf[:3])
            exec_ms.append(buf[2])
        if k == 4:
            exec_elems = int(buf[3])
    L.rs_profile(0)
    ms_step = total_ms / args.steps
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms_step], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_step = float(tt.item())
    value = n * world / (ms_step / 1e3)

    # e2e through the public API from pinned host memory
    hk = torch.from_numpy(keys_np).pin_memory()
    ht = torch.from_numpy(tags_np).pin_memory() if tags_np is not None else None
    e2e_ms = 0.0
    for it in range(args.warmup + args.steps):
        hk.copy_(torch.from_numpy(keys_np))
        if ht is not None:
            ht.copy_(torch.from_numpy(tags_np))
        flush.fill_(1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mm = rs.SORTERS[args.algo](hk, rs.SortConfig(), None, ht)
        e1.record(stream)
        e1.synchronize()
        if it >= args.warmup:
            e2e_ms += e0.elapsed_time(e1)
    e2e_step = e2e_ms / args.steps
    assert mm.merge_cost == metrics["merge_cost"]
    ok = bool(np.all(hk.numpy()[:-1] <= hk.numpy()[1:]))

    peak, peak_src = hbm_peak()
    # merge executor: every element of every merge it runs is read + written once
    alg_bytes = 2.0 * B * (exec_elems if exec_elems is not None else metrics["merge_cost"])
    whole_bytes = 2.0 * B * (metrics["merge_cost"] + n)  # + one leaf-formation pass
    exec_avg = float(np.mean(exec_ms)) if exec_ms else float("nan")
    achieved = alg_bytes / (exec_avg / 1e3) / 1e9
    whole = whole_bytes / (ms_step / 1e3) / 1e9
    traffic = None
    try:
        tj = json.load(open(os.path.join(REPO, "profiles", "traffic.json")))
        t = tj.get(f"cfg{args.config}")
        if t:
            traffic = t["dram_read_bytes"] + t["dram_write_bytes"]
    except Exception:
        pass
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "keys/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32" if kb == 4 else "int64",
        "data": "synthetic (seeded PCG64 generator, SURVEY App. B)",
        "config": {
            "workload": f"cfg{args.config}: " + ["", "perm 2^20 int32", "random-runs 1e7 int32 mean sqrt(n)",
                                                 "zipf mixed-direction 2^24 int32", "stability 1e8 int32+int32"][args.config],
            "n_per_gpu": n, "key_bytes": kb, "tag_bytes": tb, "min_run_len": 24, "merge_kind": "bitonic",
            "algo": args.algo, "l2": "flushed (512 MiB write) before every timed step",
            "parallelism": f"shard{world}" if world > 1 else "single-gpu",
        },
        "sorted_ok": ok,
        "metrics": metrics,
        "phase_ms": {k: float(v / max(1, len(exec_ms))) for k, v in zip(["prep", "phaseA", "merge"], phase)},
        "gpu_launches": KERNELS_PER_SORT * args.steps,
        "e2e": {"value": n * world / (e2e_step / 1e3), "unit": "keys/s", "ms_per_step": e2e_step,
                "h2d_bytes_per_step": n * B, "d2h_bytes_per_step": n * B + 32},
        "roofline": {"bound": "hbm", "kernel": "k_merge_exec (all merges of the large tree nodes)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": "profiles/traffic.json (ncu --set full, one launch)",
                     "algorithmic_bytes_per_launch": alg_bytes, "merged_elements_per_launch": exec_elems,
                     "whole_sort_achieved": whole, "whole_sort_frac": whole / peak, "peak_source": peak_src},
        "clocks": clk,
    }
    return out


def run_cpu_reference(args, as_baseline=False):
    keys, tags = make_input(args.config, args.n)
    threads = host_threads()
    secs = args.cpu_seconds
    v, info = cpu_oracle_throughput(keys, tags, secs, threads, args.algo)
    cpu = {"value": v, "unit": "keys/s", "cores": threads, "kind": "port",
           "sample": f"{info['sorts']} full cfg{args.config} sorts (n={len(keys)}), one per thread at a time, "
                     f"{info['wall_s']} s wall; single sort {info['single_sort_s']} s",
           "impl": "oracle/runsort_oracle.c (C restatement of reference " + args.algo + ", sorters.py:"
                   + ("430-519" if args.algo == "powersort" else "146-361") + ")"}
    return cpu


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="use the multi-GPU sharded path even at N=1")
    ap.add_argument("--algo", default="powersort", choices=["powersort", "peeksort"])
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        cpu = run_cpu_reference(args)
        keys_n = args.n or {1: 1 << 20, 2: 10**7, 3: 1 << 24, 4: 10**8}[args.config]
        out = {"impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "keys/s",
               "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": keys_n / cpu["value"] * 1e3, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
               "config": {"workload": f"cfg{args.config}", "n_per_gpu": keys_n, "algo": args.algo,
                          "min_run_len": 24, "merge_kind": "bitonic"},
               "cpu_baseline": cpu,
               "e2e": {"value": cpu["value"], "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return 0

    if (world > 1 or args.sharded) and args.algo != "powersort":
        raise SystemExit("the sharded multi-GPU path runs powersort on each shard (--algo powersort)")
    if world > 1 or args.sharded:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl")
        from paper_1805_04154_b200 import dist as rsdist

        clocks = Clocks(local_rank)
        clocks.start()
        out = rsdist.bench_sharded(args, rank, world, local_rank)
        out["clocks"] = clocks.stop()
        if rank == 0:
            if world == 1 and not args.no_cpu_baseline:
                out["cpu_baseline"] = run_cpu_reference(args)
            print(json.dumps(out))
        dist.destroy_process_group()
        return 0

    out = run_ours(args, rank, world, local_rank)
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = run_cpu_reference(args)
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
