"""``.zgla`` tensor files, byte-compatible with the reference (glasp/tensorio.py:1-49).

Format: magic ``ZGLA``, ndim as little-endian u32, each dim as little-endian u32,
then the values as little-endian float64 in C order.  GPU results (bf16/fp32
outputs and gradients, torch or NumPy) are widened to float64 on write, so a
file written here diffs directly against one the reference wrote for the same
run (``glasp.reports.export_artifacts``).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .errors import TensorFormatError

MAGIC = b"ZGLA"


def _to_numpy(values) -> np.ndarray:
    try:
        import torch
        if isinstance(values, torch.Tensor):
            return values.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(values, dtype=np.float64)


def encode_tensor(values) -> bytes:
    arr = np.asarray(_to_numpy(values), dtype="<f8")  # (ascontiguousarray would lift a 0-d array to 1-d)
    if any(d >= 2 ** 32 for d in arr.shape):
        raise TensorFormatError(f"dimension too large for a u32 header: {arr.shape}")
    head = MAGIC + struct.pack("<I", arr.ndim) + struct.pack(f"<{arr.ndim}I", *arr.shape)
    return head + arr.tobytes(order="C")


def decode_tensor(raw: bytes, name: str = "<bytes>") -> np.ndarray:
    if len(raw) < 8 or raw[:4] != MAGIC:
        raise TensorFormatError(f"{name}: missing {MAGIC!r} magic")
    (ndim,) = struct.unpack("<I", raw[4:8])
    end = 8 + 4 * ndim
    if len(raw) < end:
        raise TensorFormatError(f"{name}: truncated header")
    shape = struct.unpack(f"<{ndim}I", raw[8:end])
    count = int(np.prod(shape, dtype=np.int64)) if ndim else 1
    if len(raw) != end + 8 * count:
        raise TensorFormatError(f"{name}: expected {end + 8 * count} bytes for shape {shape}, got {len(raw)}")
    return np.frombuffer(raw, dtype="<f8", offset=end, count=count).reshape(shape).astype(np.float64)


def write_tensor(path, values) -> None:
    """glasp/tensorio.py:21-27."""
    Path(path).write_bytes(encode_tensor(values))


def read_tensor(path) -> np.ndarray:
    """glasp/tensorio.py:30-49 (same TensorFormatError cases)."""
    return decode_tensor(Path(path).read_bytes(), str(path))
