"""DWM1 tensor files: the reference's byte-exact
interchange format (``pkg/src/dwmconv/tensorfile.py:1-58``), so the reference
and the B200 path can run on identical inputs and their outputs compared
byte for byte.

    offset 0   b"DWM1"
    offset 4   u32 rank (= 4)
    offset 8   u32 N, C, H, W
    offset 24  u8 precision tag (0 = binary32, 1 = binary64)
    offset 25  payload, row-major N,C,H,W, little-endian
"""

import struct

import numpy as np

MAGIC = b"DWM1"
HEADER = struct.Struct("<4s5IB")
TAGS = {0: np.dtype("<f4"), 1: np.dtype("<f8")}


def _tag_of(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return 0
    if dt == np.float64:
        return 1
    raise TypeError(f"only binary32/binary64 tensors can be stored, got {dt}")


def write_tensor(path, tensor) -> None:
    """Write a 4-D float32/float64 array (NumPy or torch) as DWM1."""
    if hasattr(tensor, "detach"):  # torch tensor
        tensor = tensor.detach().cpu().numpy()
    if not isinstance(tensor, np.ndarray):
        raise TypeError(f"tensor must be a numpy array, got {type(tensor).__name__}")
    if tensor.ndim != 4:
        raise ValueError(f"tensor must have 4 axes (N,C,H,W), got shape {tensor.shape}")
    tag = _tag_of(tensor.dtype)
    body = np.ascontiguousarray(tensor, dtype=TAGS[tag])
    with open(path, "wb") as fh:
        fh.write(HEADER.pack(MAGIC, 4, *(int(s) for s in tensor.shape), tag))
        fh.write(memoryview(body).cast("B"))


def read_tensor(path) -> np.ndarray:
    """Read a DWM1 file into a native-endian NumPy array (ValueError on any
    malformed header or payload size, with the reference's messages)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < HEADER.size:
        raise ValueError(f"{path}: truncated header")
    magic, rank, n, c, h, w, tag = HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}, expected {MAGIC!r}")
    if rank != 4:
        raise ValueError(f"{path}: rank {rank} unsupported, expected 4")
    if tag not in TAGS:
        raise ValueError(f"{path}: unknown precision tag {tag}")
    dt = TAGS[tag]
    count = n * c * h * w
    have = len(raw) - HEADER.size
    if have != count * dt.itemsize:
        raise ValueError(f"{path}: payload is {have} bytes, expected {count * dt.itemsize}")
    arr = np.frombuffer(raw, dtype=dt, count=count, offset=HEADER.size).reshape(n, c, h, w)
    return arr.astype(dt.newbyteorder("="), copy=True)
