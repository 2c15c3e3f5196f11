"""Particle ordering and fixed-radius neighbour counts on the GPU.

``particle_perm`` is ``build_octree(positions).particle_perm`` of the
reference (octree.py:306-348): the GPU computes 63-bit x-major Morton keys
with the reference's own fp64 centre arithmetic, radix-sorts them stably,
finds each particle's capacity-8 leaf (with the coincident-point guard) and
orders particles inside a leaf by original index -- the same permutation,
bit for bit.

``neighbor_counts`` is ``range_query(tree, pos_i, h_i, exclude=i).size``
(octree.py:351-379) for every particle at once: the number of other
particles with (dx*dx + dy*dy) + dz*dz <= h_i*h_i in unfused fp64.
"""

from __future__ import annotations

import numpy as np

from . import _lib

DEFAULT_LEAF_CAPACITY = 8
MAX_TREE_DEPTH = 48


def _xyz(positions, dtype=None):
    if isinstance(positions, (tuple, list)) and len(positions) == 3:
        arrs = [np.asarray(a) for a in positions]
    else:
        pos = np.asarray(positions)
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise ValueError(f"expected an (N, 3) position array, got shape {pos.shape}")
        arrs = [pos[:, 0], pos[:, 1], pos[:, 2]]
    if dtype is None:
        dtype = np.float32 if all(a.dtype == np.float32 for a in arrs) else np.float64
    x, y, z = (np.ascontiguousarray(a, dtype=dtype) for a in arrs)
    if not (x.ndim == y.ndim == z.ndim == 1 and x.shape == y.shape == z.shape):
        raise ValueError("x, y, z must be 1-D arrays of equal length")
    return x, y, z


def particle_perm(positions, leaf_capacity: int = DEFAULT_LEAF_CAPACITY, device: int = 0) -> np.ndarray:
    """The reference octree's particle_perm (leaf capacity 8 only)."""
    if leaf_capacity != DEFAULT_LEAF_CAPACITY:
        raise ValueError("the GPU ordering implements the reference leaf capacity 8")
    x, y, z = _xyz(positions)
    n = x.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    if not (np.isfinite(x).all() and np.isfinite(y).all() and np.isfinite(z).all()):
        raise ValueError("positions must be finite")
    ctx = _lib.context(device)
    out = np.empty(n, dtype=np.int64)
    prec = _lib.PRECISION["f32" if x.dtype == np.float32 else "f64"]
    rc = _lib.load().sph_sort_perm(ctx, prec, n, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z), _lib.ptr(out))
    if rc != _lib.SPH_OK:
        msg = _lib.last_error(ctx)
        raise (ValueError if rc == _lib.SPH_INVALID else RuntimeError)(msg)
    return out


def neighbor_counts(positions, h, periodic: bool = False, box: float = 0.0, device: int = 0,
                    return_stats: bool = False):
    """#{j != i : d2_ij <= h_i^2} per particle (exact fp64 comparison)."""
    x, y, z = _xyz(positions)
    n = x.shape[0]
    hh = np.ascontiguousarray(np.broadcast_to(np.asarray(h, dtype=np.float64), (n,)))
    if n == 0:
        return np.zeros(0, dtype=np.int32)
    ctx = _lib.context(device)
    out = np.empty(n, dtype=np.int32)
    st = _lib.SphStats()
    prec = _lib.PRECISION["f32" if x.dtype == np.float32 else "auto"]
    rc = _lib.load().sph_neighbor_counts(ctx, prec, 1 if periodic else 0, float(box), n, _lib.ptr(x),
                                         _lib.ptr(y), _lib.ptr(z), _lib.ptr(hh), _lib.ptr(out), st)
    if rc != _lib.SPH_OK:
        msg = _lib.last_error(ctx)
        raise (ValueError if rc == _lib.SPH_INVALID else RuntimeError)(msg)
    return (out, st.as_dict()) if return_stats else out


def range_query_all(positions, h, device: int = 0):
    """``range_query(tree, pos_i, h_i, exclude=i)`` (octree.py:351-379) for
    every particle i at once, open boundary: CSR (offsets int64[n+1], idx
    int64[total], d2 float64[total]); each list sorted by index (the
    reference lists the same set in tree order)."""
    x, y, z = _xyz(positions)
    n = x.shape[0]
    hh = np.ascontiguousarray(np.broadcast_to(np.asarray(h, dtype=np.float64), (n,)))
    if n == 0:
        return np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0)
    counts = neighbor_counts((x, y, z), hh, device=device)
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    idx = np.empty(int(offsets[-1]), dtype=np.int64)
    d2 = np.empty(int(offsets[-1]), dtype=np.float64)
    ctx = _lib.context(device)
    prec = _lib.PRECISION["f32" if x.dtype == np.float32 else "auto"]
    rc = _lib.load().sph_range_query(ctx, prec, n, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z), _lib.ptr(hh),
                                     _lib.ptr(offsets), _lib.ptr(idx), _lib.ptr(d2))
    if rc != _lib.SPH_OK:
        msg = _lib.last_error(ctx)
        raise (ValueError if rc == _lib.SPH_INVALID else RuntimeError)(msg)
    return offsets, idx, d2
