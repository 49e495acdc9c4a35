"""Array-file fixtures written by the REFERENCE's own serializer.

    python tests/golden/make_bin.py

Imports the reference from /root/reference/pkg/src (only in this container)
and writes, with its gen.save_array (gen.py:210-222), a ".bin" and a ".txt"
file of the same seeded int64 array (extremes included), plus the expected
values as .npy.  tests/test_io.py and tests/test_gpu_io.py read them.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from runsort import gen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(1805_04154)
a = rng.integers(-(1 << 62), 1 << 62, size=3000, dtype=np.int64)
a[:4] = [np.iinfo(np.int64).min, np.iinfo(np.int64).max, 0, -1]
gen.save_array(os.path.join(HERE, "ref_array.bin"), a)
gen.save_array(os.path.join(HERE, "ref_array.txt"), a[:200])
np.save(os.path.join(HERE, "ref_array.npy"), a)
print("wrote", len(a), "values")
