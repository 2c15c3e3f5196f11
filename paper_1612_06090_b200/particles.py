"""Particle record layout of the drop-in boundary.

The host-side array format is the reference's packed record
(particles.py:20-33, 68-77 of the reference): ``id i8, x f8, y f8, z f8,
mass f8, smoothing_length f8, density f8, needs_recompute u1`` followed by an
opaque pad up to ``record_bytes`` (224 by default).  The GPU never sees this
record: the C ABI takes the base pointer plus the record stride and pulls
only x, y, z, mass and smoothing_length across PCIe (strided 2-D copies),
then writes smoothing_length, density and needs_recompute back the same way.

``ParticleSoA`` / ``gather_to_soa`` / ``scatter_from_soa`` mirror the
reference's compact-layout helpers (particles.py:87-185) for callers that
use them directly.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

LIVE_FIELDS = (
    ("id", "<i8"),
    ("x", "<f8"),
    ("y", "<f8"),
    ("z", "<f8"),
    ("mass", "<f8"),
    ("smoothing_length", "<f8"),
    ("density", "<f8"),
    ("needs_recompute", "u1"),
)
LIVE_RECORD_BYTES = 57
DEFAULT_AOS_RECORD_BYTES = 224
SOA_MAX_BYTES_PER_PARTICLE = 64
ALL_FIELDS = frozenset({"position", "mass", "smoothing_length", "density", "needs_recompute"})
DEFAULT_SCATTER_FIELDS = frozenset({"density", "smoothing_length", "needs_recompute"})

# byte offsets inside a record (used by the C ABI's strided copies)
FIELD_OFFSETS = {"id": 0, "x": 8, "y": 16, "z": 24, "mass": 32, "smoothing_length": 40,
                 "density": 48, "needs_recompute": 56}


class LayoutKind(Enum):
    AOS = "aos"
    SOA = "soa"


def _check_record_bytes(record_bytes: int) -> None:
    floor = max(64, LIVE_RECORD_BYTES)
    if record_bytes < floor:
        raise ValueError(f"aos_record_bytes must be >= {floor}, got {record_bytes}")


@dataclass(frozen=True)
class LayoutConfig:
    aos_record_bytes: int = DEFAULT_AOS_RECORD_BYTES
    layout_kind: LayoutKind = LayoutKind.AOS

    def __post_init__(self):
        _check_record_bytes(self.aos_record_bytes)


def aos_dtype(record_bytes: int = DEFAULT_AOS_RECORD_BYTES) -> np.dtype:
    """Packed structured dtype of one particle record."""
    _check_record_bytes(record_bytes)
    fields = list(LIVE_FIELDS)
    pad = record_bytes - LIVE_RECORD_BYTES
    if pad:
        fields.append(("pad", "u1", (pad,)))
    dt = np.dtype(fields)
    assert dt.itemsize == record_bytes
    return dt


def new_particle_array(n: int, record_bytes: int = DEFAULT_AOS_RECORD_BYTES) -> np.ndarray:
    if n < 0:
        raise ValueError("particle count must be non-negative")
    return np.zeros(n, dtype=aos_dtype(record_bytes))


def is_packed_record_array(particles: np.ndarray) -> bool:
    """True when ``particles`` uses the reference record layout (any size)."""
    dt = particles.dtype
    if dt.names is None:
        return False
    for name, off in FIELD_OFFSETS.items():
        if name not in dt.fields or dt.fields[name][1] != off:
            return False
    return True


@dataclass
class ParticleSoA:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    mass: np.ndarray
    smoothing_length: np.ndarray
    density: np.ndarray
    needs_recompute: np.ndarray

    BYTES_PER_PARTICLE = 6 * 8 + 1

    @property
    def count(self) -> int:
        return int(self.x.shape[0])

    @classmethod
    def empty(cls, n: int) -> "ParticleSoA":
        return cls(*(np.empty(n) for _ in range(6)), needs_recompute=np.empty(n, dtype=np.uint8))

    def validate(self) -> None:
        n = self.count
        for name in ("y", "z", "mass", "smoothing_length", "density", "needs_recompute"):
            if getattr(self, name).shape != (n,):
                raise ValueError(f"SoA field {name} has shape {getattr(self, name).shape}, "
                                 f"expected ({n},)")


def gather_to_soa(particles: np.ndarray, out: ParticleSoA | None = None,
                  start: int = 0, stop: int | None = None) -> ParticleSoA:
    n = particles.shape[0]
    stop = n if stop is None else stop
    out = ParticleSoA.empty(n) if out is None else out
    if out.count != n:
        raise ValueError(f"gather target holds {out.count} particles, source has {n}")
    sl = slice(start, stop)
    for name in ("x", "y", "z", "mass", "smoothing_length", "density", "needs_recompute"):
        getattr(out, name)[sl] = particles[name][sl]
    return out


def scatter_from_soa(soa: ParticleSoA, particles: np.ndarray,
                     fields=DEFAULT_SCATTER_FIELDS, start: int = 0,
                     stop: int | None = None) -> np.ndarray:
    if soa.count != particles.shape[0]:
        raise ValueError(f"scatter size mismatch: SoA holds {soa.count} particles, "
                         f"AoS holds {particles.shape[0]}")
    unknown = set(fields) - ALL_FIELDS
    if unknown:
        raise ValueError(f"unknown scatter fields: {sorted(unknown)}")
    sl = slice(start, soa.count if stop is None else stop)
    names = []
    for f in fields:
        names.extend(("x", "y", "z") if f == "position" else (f,))
    for name in names:
        particles[name][sl] = getattr(soa, name)[sl]
    return particles
