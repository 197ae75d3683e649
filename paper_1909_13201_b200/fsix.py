"""FSIX archive reader/writer.

FSIX is the flat container the reference-side exporter
(``oracle/ref_harness/harness.cpp``) writes: an 8-byte magic ``FSIX0001``
followed by records ``u32 name_len | name | 4-byte dtype ("f8","i4","u1")
| i64 count | raw little-endian payload``.  Used for the solve-phase inputs
(level CSR matrices in the J2 frame, transfers, masks, FS block sets) and
for golden outputs of the unmodified reference.
"""
from __future__ import annotations

import struct
from typing import Dict

import numpy as np

_MAGIC = b"FSIX0001"
_DT = {"f8": np.float64, "i4": np.int32, "u1": np.uint8}


def load(path: str) -> Dict[str, np.ndarray]:
    out: Dict[str, np.ndarray] = {}
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != _MAGIC:
        raise ValueError(f"{path}: not an FSIX archive")
    off = 8
    n = len(data)
    while off < n:
        (nl,) = struct.unpack_from("<I", data, off)
        off += 4
        name = data[off:off + nl].decode()
        off += nl
        dt = data[off:off + 4].rstrip(b"\0").decode()
        off += 4
        (count,) = struct.unpack_from("<q", data, off)
        off += 8
        dtype = np.dtype(_DT[dt])
        nbytes = count * dtype.itemsize
        out[name] = np.frombuffer(data, dtype=dtype, count=count, offset=off).copy()
        off += nbytes
    return out


def save(path: str, arrays: Dict[str, np.ndarray]) -> None:
    inv = {np.dtype(np.float64): "f8", np.dtype(np.int32): "i4", np.dtype(np.uint8): "u1"}
    with open(path, "wb") as f:
        f.write(_MAGIC)
        for name, a in arrays.items():
            a = np.ascontiguousarray(a)
            dt = inv[a.dtype]
            nb = name.encode()
            f.write(struct.pack("<I", len(nb)))
            f.write(nb)
            f.write(dt.encode().ljust(4, b"\0"))
            f.write(struct.pack("<q", a.size))
            f.write(a.tobytes())
