"""Time the REFERENCE's own powersort / peeksort (pure Python + numpy,
/root/reference/pkg/src/runsort) single-threaded on the BASELINE configs in the
build container, exactly as its harness times it (perf_counter_ns around the
call, reference bench.py:163-167).  The reference cannot travel to the GPU box,
so bench.py reports these numbers as a labelled static baseline beside the
live C-port timings.  Writes profiles/ref_python_times.json."""
import json
import os
import platform
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from runsort import Metrics, SortConfig, peeksort, powersort  # noqa: E402

from paper_1805_04154_b200 import workloads  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


out = {"what": "reference runsort.powersort / peeksort, single thread, perf_counter_ns around the call",
       "cpu_model": cpu_model(), "host_threads": os.cpu_count(), "python": sys.version.split()[0], "runs": {}}
for cfg in [int(x) for x in (sys.argv[1:] or ["1", "2", "3", "4"])]:
    keys, tags = workloads.generate(cfg)
    for name, fn in (("powersort", powersort), ("peeksort", peeksort)):
        if cfg == 4 and name == "peeksort":
            continue
        a = keys.copy()
        t = None if tags is None else tags.copy()
        m = Metrics()
        t0 = time.perf_counter_ns()
        fn(a, SortConfig(), m, t)
        dt = time.perf_counter_ns() - t0
        out["runs"][f"cfg{cfg}_{name}"] = {"n": len(keys), "seconds": dt / 1e9, "keys_per_s": len(keys) / (dt / 1e9),
                                           "metrics": [m.merge_cost, m.comparisons, m.runs_detected,
                                                       m.max_stack_height]}
        print(cfg, name, dt / 1e9, flush=True)
with open(os.path.join(REPO, "profiles", "ref_python_times.json"), "w") as fh:
    json.dump(out, fh, indent=1)
