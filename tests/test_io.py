"""Array files (reference gen.py:205-236): host parity with fixtures written by
the reference's own save_array (tests/golden/make_bin.py)."""
import os

import numpy as np
import pytest

from paper_1805_04154_b200 import io as rio

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_load_reference_files():
    want = np.load(os.path.join(G, "ref_array.npy"))
    got = rio.load_array(os.path.join(G, "ref_array.bin"))
    assert got.dtype == np.int64 and np.array_equal(got, want)
    got_t = rio.load_array(os.path.join(G, "ref_array.txt"))
    assert np.array_equal(got_t, want[:200])


def test_save_is_byte_identical(tmp_path):
    want = np.load(os.path.join(G, "ref_array.npy"))
    rio.save_array(tmp_path / "x.bin", want)
    assert (tmp_path / "x.bin").read_bytes() == open(os.path.join(G, "ref_array.bin"), "rb").read()
    rio.save_array(tmp_path / "x.txt", want[:200])
    assert (tmp_path / "x.txt").read_text() == open(os.path.join(G, "ref_array.txt")).read()


def test_unsupported_suffix(tmp_path):
    with pytest.raises(ValueError):
        rio.save_array(tmp_path / "x.csv", [1, 2])
    with pytest.raises(ValueError):
        rio.load_array(tmp_path / "x.csv")
