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

``build_octree`` / ``range_query`` mirror the reference's tree object and its
query around an arbitrary centre (octree.py:244-273, 306-379): the tree is
built once on the device (kept in its own library context) and queried any
number of times; ``range_query_many`` answers a batch of centres in one call.
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
    """The reference octree's particle_perm (build_octree(positions,
    leaf_capacity).particle_perm, octree.py:306-348), leaf capacity 1-32,
    depth up to 48."""
    if leaf_capacity < 1:
        raise ValueError(f"leaf_capacity must be >= 1, got {leaf_capacity}")
    x, y, z = _xyz(positions)
    n = x.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    if not (np.isfinite(x).all() and np.isfinite(y).all() and np.isfinite(z).all()):
        raise ValueError("positions must be finite")
    ctx = _lib.context(device)
    out = np.empty(n, dtype=np.int64)
    prec = _lib.PRECISION["f32" if x.dtype == np.float32 else "f64"]
    rc = _lib.load().sph_sort_perm_ex(ctx, prec, n, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z), int(leaf_capacity),
                                      _lib.ptr(out))
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


class QueryWorkspace:
    """Accepted for signature compatibility with the reference
    (octree.py:276-289); the device query allocates its own buffers."""

    def __init__(self, capacity: int = 2048):
        self.capacity = capacity


class Octree:
    """The reference's Octree (octree.py:244-273) as a device-resident search
    tree: positions ordered by the bit-exact octree keys, cells of <= 32
    particles with tight fp32 boxes.  ``particle_perm`` is the reference
    permutation (computed on first use); queries go through
    ``range_query`` / ``range_query_many``."""

    def __init__(self, positions, leaf_capacity: int = DEFAULT_LEAF_CAPACITY, device: int = 0):
        import ctypes
        if leaf_capacity < 1:
            raise ValueError(f"leaf_capacity must be >= 1, got {leaf_capacity}")
        x, y, z = _xyz(positions)
        if x.shape[0] and not (np.isfinite(x).all() and np.isfinite(y).all() and np.isfinite(z).all()):
            raise ValueError("positions must be finite")
        self.x, self.y, self.z = x, y, z
        self.leaf_capacity = leaf_capacity
        self.device = device
        self._perm = None
        self._ctx = None
        n = x.shape[0]
        if n == 0:
            return
        L = _lib.load()
        if L.sph_device_count() <= 0:
            raise RuntimeError("no CUDA device visible: the B200 pass has no CPU fallback")
        h = ctypes.c_void_p()
        rc = L.sph_ctx_create(ctypes.byref(h), device)
        if rc != _lib.SPH_OK:
            raise RuntimeError(f"sph_ctx_create(device={device}) failed with status {rc}")
        self._ctx = h
        prec = _lib.PRECISION["f32" if x.dtype == np.float32 else "auto"]
        rc = L.sph_octree_build(h, prec, n, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z))
        if rc != _lib.SPH_OK:
            raise (ValueError if rc == _lib.SPH_INVALID else RuntimeError)(_lib.last_error(h))

    def __del__(self):
        if getattr(self, "_ctx", None) is not None:
            try:
                _lib.load().sph_ctx_destroy(self._ctx)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
            self._ctx = None

    @property
    def n_particles(self) -> int:
        return int(self.x.shape[0])

    @property
    def particle_perm(self) -> np.ndarray:
        if self._perm is None:
            self._perm = particle_perm((self.x, self.y, self.z), self.leaf_capacity, self.device)
        return self._perm


def build_octree(positions, leaf_capacity: int = DEFAULT_LEAF_CAPACITY, max_depth: int = MAX_TREE_DEPTH,
                 device: int = 0) -> Octree:
    """``build_octree`` (octree.py:306-348) on the device."""
    if max_depth < 1:
        raise ValueError(f"max_depth must be >= 1, got {max_depth}")
    return Octree(positions, leaf_capacity, device)


def range_query_many(tree: Octree, centers, radii, exclude=None):
    """``range_query`` for many centres at once: CSR (offsets int64[m+1],
    idx int64[total], d2 float64[total]), each list sorted by index."""
    c = np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(-1, 3))
    m = c.shape[0]
    r = np.ascontiguousarray(np.broadcast_to(np.asarray(radii, dtype=np.float64), (m,)))
    if np.any(r < 0.0) or np.any(np.isnan(r)):
        bad = r[~(r >= 0.0)][0]
        raise ValueError(f"radius must be non-negative, got {bad}")
    ex = None if exclude is None else np.ascontiguousarray(
        np.broadcast_to(np.asarray(exclude, dtype=np.int64), (m,)))
    offsets = np.zeros(m + 1, dtype=np.int64)
    if tree.n_particles == 0 or m == 0:
        return offsets, np.zeros(0, dtype=np.int64), np.zeros(0)
    import ctypes
    L = _lib.load()
    total = ctypes.c_int64(0)
    cap = max(1024, 64 * m)
    while True:
        idx = np.empty(cap, dtype=np.int64)
        d2 = np.empty(cap, dtype=np.float64)
        rc = L.sph_octree_query(tree._ctx, m, _lib.ptr(c), _lib.ptr(r), _lib.ptr(ex) if ex is not None else None,
                                cap, _lib.ptr(offsets), _lib.ptr(idx), _lib.ptr(d2), ctypes.byref(total))
        if rc == _lib.SPH_INVALID and total.value > cap:
            cap = int(total.value)  # the reference's workspace.grow()
            continue
        if rc != _lib.SPH_OK:
            raise (ValueError if rc == _lib.SPH_INVALID else RuntimeError)(_lib.last_error(tree._ctx))
        t = int(total.value)
        return offsets, idx[:t], d2[:t]


def range_query(tree: Octree, center, radius: float, workspace: QueryWorkspace | None = None,
                exclude: int = -1):
    """``range_query(tree, center, radius, workspace, exclude)``
    (octree.py:351-379): every particle with (dx*dx + dy*dy) + dz*dz <=
    radius*radius (unfused fp64, dx = x_j - center_x), except ``exclude``;
    (indices, squared distances) sorted by index (the reference returns the
    same set in tree order)."""
    if radius < 0.0:
        raise ValueError(f"radius must be non-negative, got {radius}")
    _, idx, d2 = range_query_many(tree, [tuple(float(v) for v in center)], [float(radius)],
                                  None if exclude < 0 else [int(exclude)])
    return idx, d2
