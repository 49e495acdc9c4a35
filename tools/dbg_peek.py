"""Which golden peeksort cases fail, and how (debug tool)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1805_04154_b200 as rs
from tests import golden_data as G
meta, arrays = G.load()
seen = set()
for case in meta["cases"]:
    if case["algo"] != "peeksort":
        continue
    a, tags = G.case_inputs(case, arrays)
    key = (case["input"], case["w"], case["merge_kind"], tags is not None)
    try:
        w = a.copy(); tw = tags.copy() if tags is not None else None
        m = rs.peeksort(w, rs.SortConfig(min_run_len=case["w"], merge_kind=case["merge_kind"]), tags=tw)
    except Exception as e:
        print('FAIL', key, 'n', len(a), a.dtype, type(e).__name__, str(e)[:80], 'runs expected', G.metrics_of(case)[2])
