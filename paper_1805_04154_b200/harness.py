"""The reference's experiment harness (``runsort.bench``: ``run_experiment``,
``verify_bounds``, the ``sortbench`` CLI, reference bench.py:142-185 and
:190-420) driven by the device sorters.

This is an adapter, not a harness: the reference looks its sorters up in the
module-global ``SORTERS`` dict (bench.py:36, call site :159-166), so routing
the reference's own harness through the B200 path is a matter of swapping
that dict's entries for the drop-in callables of ``sorters.SORTERS`` while
the harness runs.  Everything else -- generators, rows, CSV / profile files,
bound checks, exit codes -- is the reference's own code.  The reference
package must be importable (``pip install`` of the reference, or
``PYTHONPATH=<reference>/pkg/src``).
"""
from __future__ import annotations

import contextlib
import importlib
from typing import Dict, Iterator, Optional, Sequence

from . import sorters as _sorters

__all__ = ["device_sorters", "reference_bench", "run_experiment", "main"]


def reference_bench(module: str = "runsort.bench"):
    """Import the reference harness module (raises ImportError with a hint)."""
    try:
        return importlib.import_module(module)
    except ImportError as e:  # pragma: no cover - depends on the environment
        raise ImportError(
            f"the reference harness {module!r} is not importable; install the reference package "
            "or put its pkg/src on PYTHONPATH") from e


@contextlib.contextmanager
def device_sorters(bench_module=None, table: Optional[Dict] = None) -> Iterator[None]:
    """Route ``bench_module.SORTERS`` (default: the reference harness) through
    ``table`` (default: the device ``sorters.SORTERS``) for the duration of the
    block; the reference's entries are restored afterwards."""
    bm = bench_module or reference_bench()
    table = _sorters.SORTERS if table is None else table
    saved = dict(bm.SORTERS)
    bm.SORTERS.update({k: v for k, v in table.items() if k in saved})
    try:
        yield
    finally:
        bm.SORTERS.clear()
        bm.SORTERS.update(saved)


def run_experiment(spec, bench_module=None, table: Optional[Dict] = None):
    """The reference's ``run_experiment(spec)`` with the device sorters."""
    bm = bench_module or reference_bench()
    with device_sorters(bm, table):
        return bm.run_experiment(spec)


def main(argv: Optional[Sequence[str]] = None, bench_module=None, table: Optional[Dict] = None) -> int:
    """The reference's ``sortbench`` CLI (``run`` / ``verify``) with the device sorters."""
    bm = bench_module or reference_bench()
    with device_sorters(bm, table):
        return bm.main(list(argv) if argv is not None else None)


if __name__ == "__main__":  # pragma: no cover
    raise SystemExit(main())
