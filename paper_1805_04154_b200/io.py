"""Array files of the reference's generators (gen.py:205-236), loaded straight
to the device.

`save_array` / `load_array` keep the reference's formats and semantics: ".bin"
= little-endian uint64 count + that many little-endian int64 values, ".txt" =
one decimal integer per line; other suffixes raise ValueError.  `load_array`
returns a host numpy int64 array like the reference; `load_array_device` reads a
".bin" file into a CUDA tensor through `rs_load_bin` (pinned staging, chunked
async copies; no host-side int64 array is materialized).
"""
from __future__ import annotations

import ctypes
import struct
from pathlib import Path
from typing import Sequence, Union

import numpy as np

from . import _lib


def save_array(path: Union[str, Path], a: Sequence[int]) -> None:
    """gen.py:210-222."""
    path = Path(path)
    a = np.asarray(a, dtype=np.int64)
    if path.suffix == ".bin":
        with open(path, "wb") as fh:
            fh.write(struct.pack("<Q", len(a)))
            fh.write(a.astype("<i8").tobytes())
    elif path.suffix == ".txt":
        with open(path, "w") as fh:
            for x in a:
                fh.write(f"{int(x)}\n")
    else:
        raise ValueError(f"unsupported array format: {path.suffix!r}")


def load_array(path: Union[str, Path]) -> np.ndarray:
    """gen.py:225-236 (host)."""
    path = Path(path)
    if path.suffix == ".bin":
        with open(path, "rb") as fh:
            (count,) = struct.unpack("<Q", fh.read(8))
            data = np.frombuffer(fh.read(8 * count), dtype="<i8", count=count)
        return data.astype(np.int64)
    if path.suffix == ".txt":
        with open(path) as fh:
            return np.array([int(line) for line in fh if line.strip()], dtype=np.int64)
    raise ValueError(f"unsupported array format: {path.suffix!r}")


def load_array_device(path: Union[str, Path], device=None):
    """Read a ".bin" array file into a new int64 CUDA tensor (rs_load_bin)."""
    import torch

    path = Path(path)
    if path.suffix != ".bin":
        raise ValueError(f"device loading reads .bin files only, got {path.suffix!r}")
    L = _lib.lib()
    n = ctypes.c_int64(0)
    _lib.check(L.rs_load_bin(str(path).encode(), ctypes.byref(n), None, 0, None))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    out = torch.empty(n.value, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        _lib.check(L.rs_load_bin(str(path).encode(), ctypes.byref(n), out.data_ptr() if n.value else None,
                                 n.value, ctypes.c_void_p(stream.cuda_stream)))
    return out
