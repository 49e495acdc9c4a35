"""Experiment harness and ``sortbench`` CLI over the device sorters.

Mirror of the reference harness ``runsort/bench.py`` (the caller of the sort
path, SURVEY §8(b) "Callers" and §8(f) item 1): the same ``ExperimentSpec``,
``ResultRow``, ``run_experiment``, ``verify_bounds``, CSV / profile files and
``sortbench run|verify`` command line, with the same columns, validation
errors and exit codes.  Every sort goes through this package's ``SORTERS``
(CUDA kernels behind the C ABI), so a results CSV is byte-identical to the
reference's for the same arguments except for ``time_ns``.

``time_ns`` brackets the sorter call only, as in the reference
(``bench.py:159-166``); for the host arrays this harness passes, that call
includes the host<->device copies.
"""
from __future__ import annotations

import argparse
import csv
import math
import struct
import sys
import time
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

from . import gen
from .gen import RunProfile, run_profile
from .runcore import Metrics
from .sorters import SORTERS, SortConfig

__all__ = [
    "ExperimentSpec", "ResultRow", "BoundViolation", "BoundsReport",
    "run_experiment", "verify_bounds", "entropy",
    "write_csv", "read_csv", "write_profiles", "read_profiles", "main",
]

GENERATORS = ("permutation", "random-runs", "timsort-drag", "file")

# columns in on-disk order (reference bench.py:55-59)
_CSV_FIELDS = [
    "algo", "generator", "n", "seed", "rep", "time_ns", "merge_cost",
    "comparisons", "runs_detected", "max_stack_height", "entropy_H",
    "normalized_cost",
]


@dataclass(frozen=True)
class ExperimentSpec:
    """Algorithms x generator x seeds x repetitions (reference bench.py:62-95)."""

    algorithms: tuple
    generator: str
    n: int
    mean_len: int = 1000
    run_scale: int = 32
    seeds: tuple = (1,)
    reps: int = 1
    merge_kind: str = "bitonic"
    min_run_len: int = 24
    verify: bool = False
    warmup: int = 0
    input_path: Optional[str] = None

    def __post_init__(self) -> None:
        if self.n < 0:
            raise ValueError("n must be >= 0")
        if self.reps < 1:
            raise ValueError("reps must be >= 1")
        for algo in self.algorithms:
            if algo not in SORTERS:
                raise ValueError(f"unknown algorithm {algo!r}; known: {sorted(SORTERS)}")
        if self.generator not in GENERATORS:
            raise ValueError(f"unknown generator {self.generator!r}; known: {GENERATORS}")
        if self.generator == "file" and not self.input_path:
            raise ValueError("generator 'file' needs input_path")


@dataclass(frozen=True)
class ResultRow:
    algo: str
    generator: str
    n: int
    seed: int
    rep: int
    time_ns: int
    merge_cost: int
    comparisons: int
    runs_detected: int
    max_stack_height: int
    entropy_H: float
    normalized_cost: float


def entropy(lengths: Sequence[int]) -> float:
    """Run-profile entropy sum (L/n) lg(n/L) (reference opttree.py:168-171).

    Evaluated term by term in Python floats and summed with the built-in
    ``sum`` in run order, exactly like the reference, so the CSV column is
    bit-identical; each distinct length's term is computed once.
    """
    lengths = [int(L) for L in lengths]
    if not lengths:
        raise ValueError("weight vector must have at least one leaf")
    if any(L <= 0 for L in lengths):
        raise ValueError("all weights must be positive")
    den = sum(lengths)
    term = {L: -(L / den) * math.log2(L / den) for L in set(lengths)}
    return float(sum(term[L] for L in lengths))


def _generate(spec: ExperimentSpec, seed: int) -> np.ndarray:
    if spec.generator == "permutation":
        return gen.random_permutation(spec.n, seed)
    if spec.generator == "random-runs":
        return gen.random_runs(spec.n, spec.mean_len, seed)
    if spec.generator == "timsort-drag":
        return gen.timsort_drag(spec.n, spec.run_scale)
    return gen.load_array(spec.input_path)


def _check_memory(n: int) -> None:
    """Host guard of the reference (bench.py:121-129) plus the device's share."""
    import psutil
    needed = 4 * 8 * max(n, 1)
    available = psutil.virtual_memory().available
    if needed > available:
        raise MemoryError(f"input of {n} keys needs ~{needed >> 20} MiB, "
                          f"only {available >> 20} MiB available")
    try:
        import torch
        if torch.cuda.is_available():
            free, _ = torch.cuda.mem_get_info()
            dev_needed = 3 * 8 * max(n, 1)  # keys + two scratch buffers
            if dev_needed > free:
                raise MemoryError(f"input of {n} keys needs ~{dev_needed >> 20} MiB of device "
                                  f"memory, only {free >> 20} MiB free")
    except ImportError:
        pass


def _normalized_cost(merge_cost: int, n: int, w: int) -> float:
    if n <= w:
        return 0.0
    return merge_cost / (n * math.log2(n / w))


def run_experiment(spec: ExperimentSpec):
    """Rows and per-seed run profiles in deterministic order (reference bench.py:138-185)."""
    _check_memory(spec.n)
    cfg = SortConfig(min_run_len=spec.min_run_len, merge_kind=spec.merge_kind)
    rows: list = []
    profiles: list = []
    for seed in spec.seeds:
        base = _generate(spec, seed)
        profile = run_profile(base)
        profiles.append((seed, profile))
        H = entropy(profile.lengths) if profile.r else 0.0
        for rep in range(spec.reps):
            for algo in spec.algorithms:
                sorter = SORTERS[algo]
                for _ in range(spec.warmup):
                    sorter(base.copy(), cfg, Metrics())
                work = base.copy()
                metrics = Metrics()
                t0 = time.perf_counter_ns()
                sorter(work, cfg, metrics)
                elapsed = time.perf_counter_ns() - t0
                if len(work) and not bool(np.all(work[:-1] <= work[1:])):
                    raise AssertionError(f"{algo} failed to sort the input")
                rows.append(ResultRow(
                    algo=algo, generator=spec.generator, n=len(base), seed=seed, rep=rep,
                    time_ns=elapsed, merge_cost=metrics.merge_cost,
                    comparisons=metrics.comparisons, runs_detected=metrics.runs_detected,
                    max_stack_height=metrics.max_stack_height, entropy_H=H,
                    normalized_cost=_normalized_cost(metrics.merge_cost, len(base),
                                                     spec.min_run_len)))
    return rows, profiles


# ------------------------------------------------------------------ bounds
@dataclass(frozen=True)
class BoundViolation:
    row: ResultRow
    bound: str
    limit: float
    actual: float


@dataclass(frozen=True)
class BoundsReport:
    checked: int
    violations: tuple

    @property
    def ok(self) -> bool:
        return not self.violations


def verify_bounds(rows: Sequence[ResultRow], profiles: Optional[dict] = None,
                  min_run_len: int = 1, merge_kind: str = "classic") -> BoundsReport:
    """Per-instance cost guarantees (reference bench.py:210-258; PAPER Thm 3/4).

    peeksort:  M <= Hn + 2n - (r+2),  C <= Hn + 3n - (2r+3)
    powersort: M <= Hn + 2n,          C <= Hn + 3n - r,  stack <= floor(lg n) + 1
    with a 1e-6*n tolerance on the entropy terms; rows with n <= 2 skipped.
    """
    if min_run_len != 1:
        raise ValueError("bounds hold for min_run_len == 1 only")
    if merge_kind != "classic":
        raise ValueError("comparison bounds hold for the classic merge only")
    violations: list = []
    checked = 0
    for row in rows:
        if row.algo not in ("peeksort", "powersort") or row.n <= 2:
            continue
        if profiles is not None and row.seed in profiles:
            prof = profiles[row.seed]
            H = entropy(prof.lengths)
            r = prof.r
            if prof.n != row.n:
                raise ValueError(f"profile for seed {row.seed} has n={prof.n}, row has {row.n}")
        else:
            H = row.entropy_H
            r = row.runs_detected
        n = row.n
        tol = 1e-6 * n
        if row.algo == "peeksort":
            checks = [("peeksort merge cost", H * n + 2 * n - (r + 2), row.merge_cost),
                      ("peeksort comparisons", H * n + 3 * n - (2 * r + 3), row.comparisons)]
        else:
            checks = [("powersort merge cost", H * n + 2 * n, row.merge_cost),
                      ("powersort comparisons", H * n + 3 * n - r, row.comparisons),
                      ("powersort stack height", math.floor(math.log2(n)) + 1,
                       row.max_stack_height)]
        checked += 1
        for name, limit, actual in checks:
            slack = tol if "stack" not in name else 0.0
            if actual > limit + slack:
                violations.append(BoundViolation(row, name, limit, actual))
    return BoundsReport(checked, tuple(violations))


# ------------------------------------------------------------- CSV / profiles
def write_csv(rows: Sequence[ResultRow], path) -> None:
    path = Path(path)
    try:
        with open(path, "w", newline="") as fh:
            writer = csv.writer(fh)
            writer.writerow(_CSV_FIELDS)
            for row in rows:
                writer.writerow([getattr(row, f) for f in _CSV_FIELDS])
    except OSError as exc:
        raise OSError(f"cannot write results to {path}: {exc}") from exc


def read_csv(path) -> list:
    path = Path(path)
    rows: list = []
    with open(path, newline="") as fh:
        reader = csv.DictReader(fh)
        missing = set(_CSV_FIELDS) - set(reader.fieldnames or ())
        if missing:
            raise ValueError(f"{path}: missing columns {sorted(missing)}")
        for rec in reader:
            rows.append(ResultRow(
                algo=rec["algo"], generator=rec["generator"], n=int(rec["n"]),
                seed=int(rec["seed"]), rep=int(rec["rep"]), time_ns=int(rec["time_ns"]),
                merge_cost=int(rec["merge_cost"]), comparisons=int(rec["comparisons"]),
                runs_detected=int(rec["runs_detected"]),
                max_stack_height=int(rec["max_stack_height"]),
                entropy_H=float(rec["entropy_H"]),
                normalized_cost=float(rec["normalized_cost"])))
    return rows


def write_profiles(profiles, path) -> None:
    """u64 count, then per seed (u64 seed, u64 r, r x u64 lengths), little-endian."""
    path = Path(path)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", len(profiles)))
        for seed, prof in profiles:
            fh.write(struct.pack("<QQ", seed, prof.r))
            fh.write(np.asarray(prof.lengths, dtype="<u8").tobytes())


def read_profiles(path) -> dict:
    path = Path(path)
    out: dict = {}
    with open(path, "rb") as fh:
        (count,) = struct.unpack("<Q", fh.read(8))
        for _ in range(count):
            seed, r = struct.unpack("<QQ", fh.read(16))
            lens = np.frombuffer(fh.read(8 * r), dtype="<u8", count=r)
            out[seed] = RunProfile(tuple(int(L) for L in lens))
    return out


# --------------------------------------------------------------------- CLI
def _parse_args(argv):
    parser = argparse.ArgumentParser(
        prog="sortbench", description="run-adaptive mergesort benchmarks and bound checks")
    sub = parser.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="generate inputs, sort, collect metrics")
    run.add_argument("--algo", required=True,
                     help=f"comma-separated algorithm names ({', '.join(sorted(SORTERS))})")
    run.add_argument("--gen", required=True, choices=GENERATORS)
    run.add_argument("--n", type=int, required=True)
    run.add_argument("--mean-len", type=int, default=1000)
    run.add_argument("--run-scale", type=int, default=32)
    run.add_argument("--seeds", type=int, default=1, help="use seeds 1..k (ignored with --seed-list)")
    run.add_argument("--seed-list", default=None, help="explicit comma-separated seeds")
    run.add_argument("--reps", type=int, default=1)
    run.add_argument("--min-run-len", type=int, default=24)
    run.add_argument("--merge", choices=("bitonic", "classic"), default="bitonic")
    run.add_argument("--warmup", type=int, default=3, help="untimed repetitions before measuring")
    run.add_argument("--verify-bounds", action="store_true")
    run.add_argument("--input", default=None, help="array file (.bin/.txt) for --gen file")
    run.add_argument("--out", default=None, help="CSV output path")
    run.add_argument("--profiles", default=None, help="write per-seed run profiles to this file")
    ver = sub.add_parser("verify", help="re-check bounds from a results CSV")
    ver.add_argument("--in", dest="infile", required=True)
    ver.add_argument("--profiles", required=True)
    return parser.parse_args(argv)


def _cmd_run(args) -> int:
    seeds = (tuple(int(s) for s in args.seed_list.split(","))
             if args.seed_list else tuple(range(1, args.seeds + 1)))
    spec = ExperimentSpec(
        algorithms=tuple(a.strip() for a in args.algo.split(",")), generator=args.gen,
        n=args.n, mean_len=args.mean_len, run_scale=args.run_scale, seeds=seeds,
        reps=args.reps, merge_kind=args.merge, min_run_len=args.min_run_len,
        warmup=args.warmup, input_path=args.input)
    rows, profiles = run_experiment(spec)
    if args.out:
        write_csv(rows, args.out)
        print(f"wrote {len(rows)} rows to {args.out}")
    else:
        writer = csv.writer(sys.stdout)
        writer.writerow(_CSV_FIELDS)
        for row in rows:
            writer.writerow([getattr(row, f) for f in _CSV_FIELDS])
    if args.profiles:
        write_profiles(profiles, args.profiles)
        print(f"wrote {len(profiles)} run profiles to {args.profiles}")
    if args.verify_bounds:
        if spec.min_run_len != 1 or spec.merge_kind != "classic":
            print("bound verification needs --min-run-len 1 --merge classic", file=sys.stderr)
            return 2
        report = verify_bounds(rows, dict(profiles), min_run_len=spec.min_run_len,
                               merge_kind=spec.merge_kind)
        _print_report(report)
        return 0 if report.ok else 1
    return 0


def _cmd_verify(args) -> int:
    report = verify_bounds(read_csv(args.infile), read_profiles(args.profiles))
    _print_report(report)
    return 0 if report.ok else 1


def _print_report(report: BoundsReport) -> None:
    if report.ok:
        print(f"bounds OK: {report.checked} rows, 0 violations")
    else:
        print(f"bounds FAILED: {len(report.violations)} violations in {report.checked} rows")
        for v in report.violations:
            print(f"  {v.bound}: {v.actual} > {v.limit:.3f} "
                  f"(algo={v.row.algo} n={v.row.n} seed={v.row.seed})")


def main(argv=None) -> int:
    """``sortbench`` (reference bench.py:425-441): 0 ok, 1 bound violated, 2 error."""
    args = _parse_args(sys.argv[1:] if argv is None else argv)
    try:
        if args.command == "run":
            return _cmd_run(args)
        return _cmd_verify(args)
    except (ValueError, OSError, MemoryError) as exc:
        print(f"sortbench: error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
