"""FNV-1a-64 digests used by the reference's determinism checks.

``density_checksum`` is the reference's bench checksum (bench.py:48-50 of
the reference: FNV-1a over the raw little-endian float64 density bytes,
16 hex digits).  The byte loop runs in the native library when it is loaded
(``sph_fnv1a64`` in the C ABI), else in a small numpy-chunked Python loop.
"""

from __future__ import annotations

import numpy as np

FNV_OFFSET_BASIS = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3


def fnv1a64(data) -> int:
    buf = np.frombuffer(memoryview(data), dtype=np.uint8)
    try:
        from ._lib import fnv1a64_native
        return fnv1a64_native(buf)
    except (ImportError, OSError):
        pass
    h = FNV_OFFSET_BASIS
    mask = 0xFFFFFFFFFFFFFFFF
    for b in buf.tolist():
        h = ((h ^ b) * FNV_PRIME) & mask
    return h


def density_checksum(densities: np.ndarray) -> str:
    return f"{fnv1a64(np.ascontiguousarray(densities, dtype='<f8').tobytes()):016x}"


def array_digest(arr: np.ndarray) -> str:
    return f"{fnv1a64(np.ascontiguousarray(arr).tobytes()):016x}"
