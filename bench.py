"""Benchmark: powersort keys/s on the BASELINE workload (config 2: n=1e7 int32 random-runs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C] [--algo powersort|peeksort] [--plane p2p|nccl]

One JSON line on rank 0.  A "step" is one sort of one synthetic batch.

ours, N = 1
  value     device-resident throughput: each step restores the unsorted input
            from an HBM copy and flushes L2 (a 512 MiB write) OUTSIDE the timed
            region, then times exactly the sort (CUDA events on its stream).
  e2e       the same sort through the public API with HOST buffers, copies in
            the timed region: ``powersort(pinned CPU tensor)`` (H2D from pinned
            host memory, sort, D2H of the result and the Metrics read), called
            from ``--e2e-callers`` (3) host threads at once, each on its own
            stream, like the reference arm's one sort per host thread (copies of
            one call overlap the other calls' sorts and opposite-direction
            copies); ``e2e_single_caller`` is one caller, one sort at a time;
            ``e2e_numpy`` is ``powersort(numpy array)`` -- the reference's own
            calling convention (sorters.py:430-450), pageable memory -- through
            the C ABI's host staging engine (rs_sort_host_ex).
  parity    outside the timed region, the timed path's output (keys and tags)
            and Metrics against the oracle: the C restatement of the reference
            for configs 1-4, the analytic oracle + torch's sort for config 5.
  roofline  the merge executor (the dominant kernel): algorithmic bytes
            2*B*(elements it merges) per launch over its CUDA-event time.
  cpu_baseline  the C port of the reference powersort on all host cores (one
            sort per thread), its single-thread latency, and the reference's own
            Python timing measured in the build container (static, labelled).
ours, N > 1 (``--gpus N`` re-launches itself under torch.distributed.run)
  every rank holds a contiguous shard of one global array; local powersort,
  device co-rank, and the W-way merge reading the peers' shards over NVLink
  (``--plane nccl``: sample splitters + all_to_all + the same merge).  Configs
  1-4: n keys per rank (weak scaling); config 5: the 2^31-key array split over
  the ranks (strong scaling).  Time = max over ranks.
reference the C port of the reference powersort on all host cores (the reference
  itself is pure Python and cannot travel to the GPU box), same config keys.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import ctypes
import json
import os
import platform
import socket
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

PEAKS = os.path.join(REPO, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
ALGO_CODES = {"powersort": 0, "peeksort": 1}  # rs_algo (include/runsort_b200.h)
METRIC = "powersort keys/s at n=1e7 int32 random-runs; % of HBM roofline; 1/2/4/8 GPU"
WORKLOAD = {1: "cfg1: perm 2^20 int32", 2: "cfg2: random-runs 1e7 int32 mean sqrt(n)",
            3: "cfg3: zipf mixed-direction 2^24 int32", 4: "cfg4: stability 1e8 int32+int32 payload",
            5: "cfg5: random-runs 2^31 int64 mean 2^16"}
DEFAULT_N = {1: 1 << 20, 2: 10**7, 3: 1 << 24, 4: 10**8, 5: 1 << 31}
KEY_BYTES = {1: 4, 2: 4, 3: 4, 4: 4, 5: 8}
TAG_BYTES = {1: 0, 2: 0, 3: 0, 4: 4, 5: 0}


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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def config_dict(args, n_per_gpu, world):
    """The `config` object both arms print (same keys => same_config)."""
    strong = args.config == 5
    return {
        "workload": WORKLOAD[args.config],
        "n_per_gpu": n_per_gpu,
        "n_total": n_per_gpu * world if not strong else DEFAULT_N[5] if args.n is None else args.n,
        "key_bytes": KEY_BYTES[args.config], "tag_bytes": TAG_BYTES[args.config],
        "min_run_len": 24, "merge_kind": "bitonic", "algo": args.algo,
        "l2": "flushed (512 MiB write) before every timed step",
        "parallelism": (f"shard{world}-{args.plane}" if world > 1 else "single-gpu"),
    }


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
    """The C port of the reference powersort / peeksort on `threads` host
    threads, each sorting its own copies of the workload for ~`seconds`."""
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
    return done * len(keys) / wall, dict(sorts=done, threads=threads, wall_s=round(wall, 3),
                                         single_sort_s=round(single, 4))


def python_reference_times():
    try:
        with open(os.path.join(REPO, "profiles", "ref_python_times.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


def run_cpu_reference(args, keys=None, tags=None):
    if keys is None:
        keys, tags = make_host_input(args.config, args.n)
    threads = host_threads()
    v, info = cpu_oracle_throughput(keys, tags, args.cpu_seconds, threads, args.algo)
    cpu = {"value": v, "unit": "keys/s", "cores": threads, "kind": "port",
           "sample": f"{info['sorts']} full cfg{args.config} sorts (n={len(keys)}), one per thread at a time, "
                     f"{info['wall_s']} s wall",
           "single_thread": {"seconds_per_sort": info["single_sort_s"],
                             "keys_per_s": len(keys) / info["single_sort_s"]},
           "cpu_model": cpu_model(),
           "impl": "oracle/runsort_oracle.c (C restatement of reference " + args.algo + ", sorters.py:"
                   + ("430-519" if args.algo == "powersort" else "146-361") + ")"}
    ref = python_reference_times()
    if ref:
        r = ref["runs"].get(f"cfg{args.config}_{args.algo}")
        if r and r["n"] == len(keys):
            cpu["python_reference"] = {
                "keys_per_s": r["keys_per_s"], "seconds_per_sort": r["seconds"], "cores": 1,
                "measured": "build container (no GPU), " + ref["cpu_model"],
                "what": "the reference's own runsort." + args.algo + " (pure Python + numpy), single thread, "
                        "perf_counter_ns around the call (reference bench.py:163-167); static, not re-timed here",
            }
    return cpu


# ------------------------------------------------------------ workloads
def make_host_input(cfg: int, n=None, seed=1):
    from paper_1805_04154_b200 import workloads

    if cfg == 5:
        raise ValueError("config 5 is generated on the device")
    return workloads.generate(cfg, n, seed)


def parity_oracle(args, keys_np, tags_np, out_k, out_t, metrics):
    """Outside the timed region: the timed path's output vs the oracle."""
    from oracle import oracle

    rk = keys_np.copy()
    rt = None if tags_np is None else tags_np.copy()
    res = getattr(oracle, args.algo)(rk, 24, "bitonic", rt)
    ok_k = bool(np.array_equal(out_k, rk))
    ok_t = True if rt is None else bool(np.array_equal(out_t, rt))
    ok_m = tuple(metrics[k] for k in ("merge_cost", "comparisons", "runs_detected", "max_stack_height")) == \
        res.metrics_tuple()
    return {"ok": ok_k and ok_t and ok_m, "keys": ok_k, "tags": ok_t, "metrics": ok_m,
            "oracle": "oracle/runsort_oracle.c on the same input"}


def parity_config5(src, out, metrics):
    """Config 5: analytic Metrics of the reference from the original array's run
    structure (oracle/analytic.py, node powers by the reference's node_power_def
    loop), the output sorted and a permutation of the input (multiset hash)."""
    import torch

    from oracle import analytic

    n = src.numel()
    asc = src[:-1] <= src[1:]
    k = torch.nonzero(asc[1:] != asc[:-1]).flatten() + 1
    bounds = torch.cat([k, torch.tensor([n - 1], device=src.device)]).cpu().numpy()
    del k
    res = analytic.powersort_metrics(
        n, 24, bounds,
        lambda pos: asc[torch.from_numpy(np.asarray(pos, dtype=np.int64)).to(src.device)].cpu().numpy(),
        lambda lo, hi: src[lo: hi + 1].cpu().numpy())
    del asc
    ok_m = tuple(metrics[k] for k in ("merge_cost", "comparisons", "runs_detected", "max_stack_height")) == \
        (res["merge_cost"], res["comparisons"], res["runs_detected"], res["max_stack_height"])
    ok_sorted = bool((out[1:] >= out[:-1]).all().item())
    ok_perm = _mix_sum(src) == _mix_sum(out)
    return {"ok": ok_m and ok_sorted and ok_perm, "metrics": ok_m, "sorted": ok_sorted, "multiset": ok_perm,
            "oracle": "oracle/analytic.py (reference powersort driver over the run structure) + "
                      "sortedness + 64-bit multiset hash"}


def _mix_sum(t):
    """Order-independent 64-bit hash of a device int tensor (sum of mixed keys)."""
    import torch

    acc = 0
    for c in range(0, t.numel(), 1 << 27):
        x = t[c: c + (1 << 27)].to(torch.int64)
        x = (x ^ (x >> 31)) * 0x5851F42D4C957F2D
        x = x ^ (x >> 29)
        acc = (acc + int(x.sum(dtype=torch.int64).item())) & ((1 << 64) - 1)
    return acc


# ------------------------------------------------------------ N = 1
def concurrent_e2e(torch, rs, algo, keys_np, tags_np, callers, per_thread):
    """Throughput of the public API with ``callers`` host threads, each sorting
    its own pinned host arrays on its own stream -- the shape of the reference
    arm (one sort per host thread).  Every sort is one synchronous
    ``powersort(pinned CPU tensor)`` call: H2D, sort, D2H and the Metrics read.
    The inputs are prepared before the timed region; the time is the host wall
    clock from the threads' common start to the last thread's last return.
    Returns (ms per sort, sorts, all outputs equal to ``ref``)."""
    import threading

    bar = threading.Barrier(callers + 1)
    t_end = [0.0] * callers
    outs = [None] * callers
    errs = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            kb = [torch.from_numpy(keys_np).pin_memory() for _ in range(per_thread + 1)]
            tb = [torch.from_numpy(tags_np).pin_memory() for _ in range(per_thread + 1)] \
                if tags_np is not None else [None] * (per_thread + 1)
            with torch.cuda.stream(s):
                rs.SORTERS[algo](kb[per_thread], rs.SortConfig(), None, tb[per_thread])  # warm-up
                bar.wait()
                for it in range(per_thread):
                    rs.SORTERS[algo](kb[it], rs.SortConfig(), None, tb[it])
                t_end[i] = time.perf_counter()
            outs[i] = (kb[:per_thread], tb[:per_thread])
        except Exception as ex:  # noqa: BLE001
            errs.append(repr(ex))
            bar.abort()

    th = [threading.Thread(target=worker, args=(i,)) for i in range(callers)]
    for t in th:
        t.start()
    try:
        bar.wait()
    except threading.BrokenBarrierError:
        pass
    t0 = time.perf_counter()
    for t in th:
        t.join()
    if errs:
        raise RuntimeError("concurrent e2e: " + "; ".join(errs))
    sorts = callers * per_thread
    return (max(t_end) - t0) * 1e3 / sorts, sorts, outs


def run_ours(args):
    import torch

    import paper_1805_04154_b200 as rs
    from paper_1805_04154_b200 import _lib, workloads

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    L = _lib.lib()
    algo = ALGO_CODES[args.algo]
    if args.config == 5:
        n = args.n or DEFAULT_N[5]
        src = workloads.config5_device(n, seed=1)
        tsrc = None
        keys_np = tags_np = None
    else:
        keys_np, tags_np = make_host_input(args.config, args.n)
        n = len(keys_np)
        src = torch.from_numpy(keys_np).to(dev)
        tsrc = torch.from_numpy(tags_np).to(dev) if tags_np is not None else None
    kb = src.element_size()
    tb = tsrc.element_size() if tsrc is not None else 0
    B = kb + tb
    work = torch.empty_like(src)
    twork = torch.empty_like(tsrc) if tsrc is not None else None
    key_code = _lib.RS_KEY_I32 if kb == 4 else _lib.RS_KEY_I64
    ws_bytes = L.rs_workspace_bytes(algo, key_code, tb, n, 24)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def one_sort(out=None):
        return L.rs_sort(algo, key_code, work.data_ptr(), tb, twork.data_ptr() if twork is not None else None,
                         n, 24, 0, ws.data_ptr(), ws_bytes, stream.cuda_stream,
                         ctypes.byref(out) if out is not None else None, None)

    def restore():
        work.copy_(src)
        if twork is not None:
            twork.copy_(tsrc)
        flush.fill_(1)

    # the correctness run (its output is checked against the oracle below)
    restore()
    m = _lib.RsMetrics()
    _lib.check(one_sort(out=m))
    metrics = dict(merge_cost=int(m.merge_cost), comparisons=int(m.comparisons),
                   runs_detected=int(m.runs_detected), max_stack_height=int(m.max_stack_height))
    if args.config == 5:
        parity = parity_config5(src, work, metrics) if args.algo == "powersort" else {"ok": None}
    else:
        parity = parity_oracle(args, keys_np, tags_np, work.cpu().numpy(),
                               twork.cpu().numpy() if twork is not None else None, metrics)

    L.rs_profile(0)  # the timed steps carry no phase events (kernels launch back to back)
    for _ in range(args.warmup):
        restore()
        _lib.check(one_sort())
    torch.cuda.synchronize()
    clocks = Clocks(0)
    clocks.start()
    time.sleep(0.3)
    times = []
    torch.cuda.synchronize()
    for _ in range(args.steps):
        restore()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(one_sort())
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    clk = clocks.stop()
    # phase split and the merge kernel's own time (roofline): the same steps
    # again with CUDA events between the kernels, outside the timed total
    phase = np.zeros(3)
    exec_ms, exec_elems = [], None
    buf = (ctypes.c_double * 4)()
    L.rs_profile(1)
    for _ in range(args.steps):
        restore()
        _lib.check(one_sort())
        torch.cuda.synchronize()
        k = L.rs_profile_read(buf, 4)
        if k >= 3:
            phase += np.array(buf[:3])
            exec_ms.append(buf[2])
        if k == 4:
            exec_elems = int(buf[3])
    L.rs_profile(0)
    ms_step = float(np.mean(times))
    value = n / (ms_step / 1e3)

    # e2e through the public API, host buffers, copies inside the timed region
    e2e_steps = args.steps if args.config != 5 else min(args.steps, 3)
    e2e_warm = args.warmup if args.config != 5 else 1
    if keys_np is None:  # config 5: the host copy of the device-generated input
        keys_np = src.cpu().numpy()
    base_k = keys_np
    base_t = tags_np
    hk_np = keys_np.copy()
    ht_np = tags_np.copy() if tags_np is not None else None
    np_ms = []
    for it in range(e2e_warm + e2e_steps):
        np.copyto(hk_np, base_k)
        if ht_np is not None:
            np.copyto(ht_np, base_t)
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mm = rs.SORTERS[args.algo](hk_np, rs.SortConfig(), None, ht_np)  # numpy in, numpy out
        dt = (time.perf_counter() - t0) * 1e3
        if it >= e2e_warm:
            np_ms.append(dt)
    assert mm.merge_cost == metrics["merge_cost"]
    e2e_np_ok = bool(np.array_equal(hk_np, work.cpu().numpy())) and \
        (ht_np is None or bool(np.array_equal(ht_np, twork.cpu().numpy())))
    hk = torch.from_numpy(keys_np).pin_memory()
    ht = torch.from_numpy(tags_np).pin_memory() if tags_np is not None else None
    pin_ms = []
    for it in range(e2e_warm + e2e_steps):
        hk.copy_(torch.from_numpy(base_k))
        if ht is not None:
            ht.copy_(torch.from_numpy(base_t))
        flush.fill_(1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mm = rs.SORTERS[args.algo](hk, rs.SortConfig(), None, ht)
        e1.record(stream)
        e1.synchronize()
        if it >= e2e_warm:
            pin_ms.append(e0.elapsed_time(e1))
    e2e_pin_ok = bool(torch.equal(hk, work.cpu())) and (ht is None or bool(torch.equal(ht, twork.cpu())))
    e2e_np = float(np.mean(np_ms))
    e2e_pin = float(np.mean(pin_ms))
    # concurrent callers (skipped when their pinned inputs would pass ~6 GB: config 5)
    callers = max(1, args.e2e_callers)
    per_thread = max(2, min(e2e_steps, int(6e9 // (callers * n * B))))
    conc = None
    if callers > 1 and callers * (per_thread + 1) * n * B <= 8e9:
        conc_ms, conc_sorts, conc_outs = concurrent_e2e(torch, rs, args.algo, base_k, base_t, callers, per_thread)
        want_k = work.cpu()
        want_t = twork.cpu() if twork is not None else None
        conc_ok = all(torch.equal(k, want_k) for ks, _ in conc_outs for k in ks) and \
            (want_t is None or all(torch.equal(t, want_t) for _, ts in conc_outs for t in ts))
        conc = {"value": n / (conc_ms / 1e3), "unit": "keys/s", "ms_per_step": conc_ms,
                "h2d_bytes_per_step": n * B, "d2h_bytes_per_step": n * B, "callers": callers,
                "sorts": conc_sorts,
                "path": f"{callers} host threads, each calling powersort(pinned CPU tensor) through the public "
                        "API on its own stream (H2D, sort, D2H, Metrics read per call) -- the reference arm's "
                        "one-sort-per-host-thread shape; inputs prepared before, host wall clock from the "
                        "common start to the last return, divided by the number of sorts",
                "output_ok": bool(conc_ok)}

    e2e_single = {"value": n / (e2e_pin / 1e3), "unit": "keys/s", "ms_per_step": e2e_pin,
                  "h2d_bytes_per_step": n * B, "d2h_bytes_per_step": n * B, "callers": 1,
                  "path": "powersort(pinned CPU tensor) through the public API, one caller: async H2D from "
                          "pinned host memory, sort, D2H of the sorted keys and the Metrics read (CUDA events "
                          "around the call)",
                  "output_ok": e2e_pin_ok}
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
    return {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32" if kb == 4 else "int64",
        "data": "synthetic (seeded PCG64 generator, SURVEY App. B)",
        "config": config_dict(args, n, 1),
        "parity": parity,
        "metrics": metrics,
        "phase_ms": {k: float(v / max(1, len(exec_ms))) for k, v in zip(["prep", "phaseA", "merge"], phase)},
        "gpu_launches": 3 * args.steps,
        "e2e": conc if conc is not None else e2e_single,
        "e2e_single_caller": e2e_single,
        "e2e_numpy": {"value": n / (e2e_np / 1e3), "unit": "keys/s", "ms_per_step": e2e_np,
                "h2d_bytes_per_step": n * B, "d2h_bytes_per_step": n * B,
                "path": "powersort(numpy array) -> rs_sort_host_ex: chunked multi-threaded pinned staging, "
                        "H2D + sort + D2H inside the timed region (host wall clock around the synchronous call)",
                "output_ok": e2e_np_ok},
        "roofline": {"bound": "hbm", "kernel": "k_merge_exec (all merges of the large tree nodes)",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": "profiles/traffic.json (ncu --set full, one launch)",
                     "algorithmic_bytes_per_launch": alg_bytes, "merged_elements_per_launch": exec_elems,
                     "whole_sort_achieved": whole, "whole_sort_frac": whole / peak, "peak_source": peak_src},
        "clocks": clk,
        "_host_inputs": (keys_np, tags_np) if args.config != 5 else None,
    }


# ------------------------------------------------------------ N > 1
def run_sharded(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1805_04154_b200 import dist as rsd
    from paper_1805_04154_b200 import workloads

    dev = torch.device("cuda", local_rank)
    if args.config == 5:  # strong scaling: one 2^31-key array split over the ranks
        n_total = args.n or DEFAULT_N[5]
        lo, hi = rank * n_total // world, (rank + 1) * n_total // world
        src = workloads.config5_range(lo, hi, n_total, seed=1, device=dev)
        tsrc = None
    else:  # weak scaling: n keys per rank, rank i's shard from seed 1 + i
        k, t = make_host_input(args.config, args.n, seed=1 + rank)
        src = torch.from_numpy(k).to(dev)
        tsrc = torch.from_numpy(t).to(dev) if t is not None else None
    n = src.numel()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    caps = [None] * world
    dist.all_gather_object(caps, n)
    cap = max(caps)
    space = None
    out_k = torch.empty(n, dtype=src.dtype, device=dev)
    out_t = torch.empty(n, dtype=tsrc.dtype, device=dev) if tsrc is not None else None
    if args.plane == "p2p":
        space = rsd.P2PShardSpace(cap, src.dtype, tsrc.dtype if tsrc is not None else None)

    def step():
        if space is not None:
            return rsd.sharded_sort_p2p(space, n, out_keys=out_k, out_tags=out_t)
        kk = work_k
        return rsd.sharded_sort(kk, work_t)

    work_k = work_t = None
    times = []
    for it in range(args.warmup + args.steps):
        if space is not None:
            space.keys[:n].copy_(src)
            if tsrc is not None:
                space.tags[:n].copy_(tsrc)
        else:
            work_k = src.clone()
            work_t = tsrc.clone() if tsrc is not None else None
        flush.fill_(1)
        torch.cuda.synchronize()
        dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ok_, ot_, info = step()
        e1.record()
        torch.cuda.synchronize()
        if it >= args.warmup:
            times.append(e0.elapsed_time(e1))
    tmax = torch.tensor([float(np.mean(times))], device=dev)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    # parity: every slice sorted, slices ordered across ranks, multiset preserved
    ok_sorted = bool((ok_[1:] >= ok_[:-1]).all().item()) if ok_.numel() > 1 else True
    edge = torch.tensor([ok_[0].item() if n else 0, ok_[-1].item() if n else 0], dtype=torch.int64, device=dev)
    edges = [torch.zeros_like(edge) for _ in range(world)]
    dist.all_gather(edges, edge)
    for i in range(world - 1):
        ok_sorted &= bool(edges[i][1].item() <= edges[i + 1][0].item())
    hs = torch.tensor([_mix_sum(src), _mix_sum(ok_)], dtype=torch.float64, device=dev)
    hsl = [torch.zeros_like(hs) for _ in range(world)]
    dist.all_gather(hsl, hs)
    hin = sum(int(x[0].item()) for x in hsl) & ((1 << 64) - 1)
    hout = sum(int(x[1].item()) for x in hsl) & ((1 << 64) - 1)
    # e2e: this rank's shard from pinned host memory, the sharded sort, its slice back
    hk = src.cpu().pin_memory()
    ht = tsrc.cpu().pin_memory() if tsrc is not None else None
    e2e = []
    for it in range(args.warmup + min(args.steps, 5)):
        flush.fill_(1)
        torch.cuda.synchronize()
        dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if space is not None:
            space.keys[:n].copy_(hk, non_blocking=True)
            if ht is not None:
                space.tags[:n].copy_(ht, non_blocking=True)
        else:
            work_k = hk.to(dev, non_blocking=True)
            work_t = ht.to(dev, non_blocking=True) if ht is not None else None
        o2, t2, _ = step()
        hk.copy_(o2, non_blocking=True)
        if t2 is not None:
            ht.copy_(t2, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        if it >= args.warmup:
            e2e.append(e0.elapsed_time(e1))
    te = torch.tensor([float(np.mean(e2e))], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    if space is not None:
        space.close()
    kb = src.element_size()
    B = kb + (tsrc.element_size() if tsrc is not None else 0)
    n_all = sum(caps)
    return {
        "metric": METRIC, "value": n_all / (ms / 1e3), "unit": "keys/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if args.config == 5 else "weak", "vs_baseline": None,
        "dtype": "int32" if kb == 4 else "int64",
        "data": "synthetic (seeded PCG64; cfg5: one array, identical for every N; cfg1-4: shard i from seed 1+i)",
        "config": config_dict(args, n, world),
        "parity": {"ok": ok_sorted and hin == hout, "sorted_across_ranks": ok_sorted, "multiset": hin == hout,
                   "oracle": "global sortedness + 64-bit multiset hash (bit-exact keys for keys-only configs)"},
        "e2e": {"value": n_all / (e2e_ms / 1e3), "unit": "keys/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": n_all * B, "d2h_bytes_per_step": n_all * B},
        # per rank per step: local powersort (3), co-rank + pivots + merge (3); NCCL plane: 3 + 2
        "gpu_launches": (6 if args.plane == "p2p" else 5) * args.steps,
    }


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="the multi-GPU path even at N=1")
    ap.add_argument("--plane", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--algo", default="powersort", choices=["powersort", "peeksort"])
    ap.add_argument("--e2e-callers", type=int, default=3,
                    help="host threads calling the public API concurrently in the e2e leg (1: single caller)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        n = args.n or DEFAULT_N[args.config]
        n_per = n // world if args.config == 5 else n
        cpu = run_cpu_reference(args) if args.config != 5 else run_cpu_reference_cfg5(args)
        out = {"impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "keys/s",
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": n_per / cpu["value"] * 1e3, "higher_is_better": True,
               "scaling": "strong" if args.config == 5 else "weak", "vs_baseline": None,
               "dtype": "int32" if KEY_BYTES[args.config] == 4 else "int64", "data": "synthetic",
               "config": config_dict(args, n_per, world),
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
        # stdout carries the one JSON line: anything a library writes to file
        # descriptor 1 while the ranks run (NCCL prints a "NCCL version ..."
        # banner there on this image) goes to stderr instead
        sys.stdout.flush()
        json_fd = os.dup(1)
        os.dup2(2, 1)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        clocks = Clocks(local_rank)
        clocks.start()
        out = run_sharded(args, rank, world, local_rank)
        out["clocks"] = clocks.stop()
        if rank == 0:
            if world == 1 and not args.no_cpu_baseline and args.config != 5:
                out["cpu_baseline"] = run_cpu_reference(args)
            os.write(json_fd, (json.dumps(out) + "\n").encode())
        dist.destroy_process_group()
        return 0

    out = run_ours(args)
    host_inputs = out.pop("_host_inputs")
    if not args.no_cpu_baseline:
        if args.config == 5:
            out["cpu_baseline"] = run_cpu_reference_cfg5(args)
        else:
            out["cpu_baseline"] = run_cpu_reference(args, *host_inputs)
    print(json.dumps(out))
    return 0


def run_cpu_reference_cfg5(args):
    """Config 5 is 16 GiB: the C port times a bounded sample of the same
    workload (its first 2^24 keys, same generator) on every host thread."""
    from paper_1805_04154_b200 import workloads

    n_s = 1 << 24
    keys = workloads.config5_range(0, n_s, DEFAULT_N[5], seed=1, device="cuda").cpu().numpy()
    cpu = run_cpu_reference(args, keys, None)
    cpu["sample"] = "first 2^24 keys of the config-5 array (same generator), " + cpu["sample"]
    return cpu


if __name__ == "__main__":
    sys.exit(main())
