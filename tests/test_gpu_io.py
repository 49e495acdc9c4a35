"""rs_load_bin: reference ".bin" files (gen.py:210-236) straight to the device."""
import os

import numpy as np
import pytest

from paper_1805_04154_b200 import io as rio

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_device_load_matches_reference_file():
    want = np.load(os.path.join(G, "ref_array.npy"))
    t = rio.load_array_device(os.path.join(G, "ref_array.bin"))
    assert t.is_cuda and str(t.dtype) == "torch.int64"
    assert np.array_equal(t.cpu().numpy(), want)


def test_device_load_large_chunked(tmp_path):
    # larger than one 32 MiB staging chunk: exercises the double-buffered path
    a = np.random.default_rng(7).integers(-(1 << 63), (1 << 63) - 1, size=(9 << 20) + 5, dtype=np.int64)
    rio.save_array(tmp_path / "big.bin", a)
    t = rio.load_array_device(tmp_path / "big.bin")
    assert np.array_equal(t.cpu().numpy(), a)


def test_device_load_then_sort(tmp_path):
    import paper_1805_04154_b200 as rs
    a = np.random.default_rng(3).integers(0, 1000, size=50_000, dtype=np.int64)
    rio.save_array(tmp_path / "s.bin", a)
    t = rio.load_array_device(tmp_path / "s.bin")
    rs.powersort(t)
    assert np.array_equal(t.cpu().numpy(), np.sort(a, kind="stable"))


def test_device_load_errors(tmp_path):
    with pytest.raises(OSError):
        rio.load_array_device(tmp_path / "missing.bin")
    bad = tmp_path / "trunc.bin"
    bad.write_bytes(np.array([10], dtype="<u8").tobytes() + np.arange(3, dtype="<i8").tobytes())
    with pytest.raises(ValueError):
        rio.load_array_device(bad)
    with pytest.raises(ValueError):
        rio.load_array_device(tmp_path / "x.txt")
