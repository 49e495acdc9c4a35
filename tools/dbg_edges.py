import sys, numpy as np
sys.path.insert(0, '.')
import paper_1805_04154_b200 as rs
from oracle import oracle
for n in [4096, 4097, 9000]:
    cases = {
        'zeros': np.zeros(n, dtype=np.int64),
        'desc': np.arange(n, 0, -1).astype(np.int64),
        'sorted': np.arange(n).astype(np.int64),
        'zigzag': (np.arange(n) % 2).astype(np.int64),
        'halves': np.concatenate([np.arange(n // 2, n), np.arange(n // 2)]).astype(np.int64),
    }
    for name, a in cases.items():
        for w in (1, 24, 1024):
            for tagged in (False, True):
                tags = np.arange(n, dtype=np.int64) if tagged else None
                ra = a.copy(); rt = None if tags is None else tags.copy()
                ref = oracle.powersort(ra, w, "classic", rt)
                wa = a.copy(); wt = None if tags is None else tags.copy()
                try:
                    m = rs.powersort(wa, rs.SortConfig(min_run_len=w, merge_kind="classic"), tags=wt)
                    got = (m.merge_cost, m.comparisons, m.runs_detected, m.max_stack_height)
                except Exception as e:
                    got = repr(e)[:80]
                ok = got == ref.metrics_tuple() and np.array_equal(wa, ra)
                if not ok:
                    print(n, name, w, tagged, got, ref.metrics_tuple(), np.array_equal(wa, ra))
print("done")
