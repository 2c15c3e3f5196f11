"""CPU oracle for the SPH density pass -- TEST INFRASTRUCTURE, NOT PRODUCT.

ctypes front end of ``sph_oracle.c`` (a plain-C restatement of the reference
``sphlab`` pass; see that file's header for the reference lines it follows)
plus a few numpy helpers.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``) may import
this package, and only as the checker / the timed CPU baseline.  The product
package ``paper_1612_06090_b200`` never imports it.

Pinning: ``tests/test_oracle_golden.py`` checks every entry point bit-for-bit
against vectors produced by the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsph_oracle.so")
_lib = None

ST_OK, ST_NOT_CONVERGED, ST_DEGENERATE, ST_INVALID = 0, 1, 2, 3

H_GROWTH = 2.0 ** (1.0 / 3.0)
WENDLAND_C6_NORM = 1365.0 / (64.0 * math.pi)


class OracleConvergenceError(RuntimeError):
    pass


class OracleDegenerateError(RuntimeError):
    pass


def build() -> str:
    """Compile the oracle shared library (idempotent)."""
    src = os.path.join(_HERE, "sph_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.sph_oracle_perm.argtypes = [i64, p, p, p, i64, p, p]
        L.sph_oracle_counts.argtypes = [i64, p, p, p, p, p, ctypes.c_int]
        L.sph_oracle_density_pass.argtypes = [i64, p, p, p, p, p, p, p, i64, i64,
                                              ctypes.c_int, p, i64, p, i64, p]
        L.sph_oracle_tree_new.argtypes = [i64, p, p, p, ctypes.POINTER(ctypes.c_int)]
        L.sph_oracle_tree_new.restype = p
        L.sph_oracle_tree_free.argtypes = [p]
        L.sph_oracle_density_pass_tree.argtypes = [p, p, p, p, p, i64, i64, ctypes.c_int, p, i64, p, i64, p]
        L.sph_oracle_w.argtypes = [ctypes.c_double, ctypes.c_double]
        L.sph_oracle_w.restype = ctypes.c_double
        L.sph_oracle_nthreads.restype = ctypes.c_int
        _lib = L
    return _lib


def _f8(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def nthreads() -> int:
    return int(lib().sph_oracle_nthreads())


def perm(x, y, z, leaf_capacity: int = 8) -> np.ndarray:
    """Octree.particle_perm of build_octree((x, y, z), leaf_capacity)."""
    x, y, z = _f8(x), _f8(y), _f8(z)
    out = np.empty(x.shape[0], dtype=np.int64)
    nn = ctypes.c_int64(0)
    st = lib().sph_oracle_perm(x.shape[0], _ptr(x), _ptr(y), _ptr(z), leaf_capacity,
                               _ptr(out), ctypes.byref(nn))
    if st:
        raise ValueError(f"oracle perm failed with status {st}")
    return out


def counts(x, y, z, h, threads: int = 0) -> np.ndarray:
    """#{j != i : (dx*dx + dy*dy) + dz*dz <= h_i*h_i} (range_query size)."""
    x, y, z, h = _f8(x), _f8(y), _f8(z), _f8(h)
    out = np.empty(x.shape[0], dtype=np.int32)
    st = lib().sph_oracle_counts(x.shape[0], _ptr(x), _ptr(y), _ptr(z), _ptr(h),
                                 _ptr(out), threads)
    if st:
        raise ValueError(f"oracle counts failed with status {st}")
    return out


class OracleResult:
    def __init__(self, h, rho, flags, todo_sizes, iterations, candidates):
        self.h = h
        self.rho = rho
        self.flags = flags
        self.todo_sizes = todo_sizes
        self.iterations = iterations
        self.candidates = candidates


def density_pass(x, y, z, mass, h0, k: int, max_iterations: int = 100,
                 threads: int = 0, targets=None) -> OracleResult:
    """The reference pass (compute_density_pass semantics) on SoA inputs.

    ``targets``: optional index subset (sampled-oracle mode); results are
    only meaningful at those indices.
    """
    x, y, z, m = _f8(x), _f8(y), _f8(z), _f8(mass)
    n = x.shape[0]
    h = _f8(h0).copy()
    rho = np.zeros(n, dtype=np.float64)
    flags = np.zeros(n, dtype=np.uint8)
    todo = np.zeros(max(max_iterations, 1) + 1, dtype=np.int64)
    info = np.zeros(4, dtype=np.int64)
    if targets is not None:
        tg = np.ascontiguousarray(targets, dtype=np.int64)
        tptr, nt = _ptr(tg), tg.shape[0]
    else:
        tptr, nt = None, n
    st = lib().sph_oracle_density_pass(n, _ptr(x), _ptr(y), _ptr(z), _ptr(m), _ptr(h),
                                       _ptr(rho), _ptr(flags), k, max_iterations,
                                       threads, tptr, nt, _ptr(todo), todo.shape[0],
                                       _ptr(info))
    if st == ST_NOT_CONVERGED:
        raise OracleConvergenceError(
            f"{int(info[2])} of {n} particles still flagged after {max_iterations} iterations")
    if st == ST_DEGENERATE:
        raise OracleDegenerateError(
            f"particle {int(info[1])}: {k}-th nearest neighbour is at zero distance; "
            f">= {k + 1} coincident particles")
    if st:
        raise ValueError(f"oracle density pass failed with status {st}")
    it = int(info[0])
    return OracleResult(h, rho, flags, todo[:it].copy(), it, int(info[3]))


class Prepared:
    """The oracle's octree over a fixed particle set, built once and reused by
    passes over target subsets (the CPU baseline's sampled timing: the tree
    build is the fixed part of a pass, timed once).  Periodic boxes: the
    originals plus their images within ``margin`` (``periodic_images``);
    targets index the originals."""

    def __init__(self, x, y, z, box: float | None = None, margin: float | None = None):
        x, y, z = _f8(x), _f8(y), _f8(z)
        self.n = x.shape[0]
        if box:
            ax, ay, az, src = periodic_images(x, y, z, box, margin if margin is not None else 0.5 * box)
        else:
            ax, ay, az, src = x, y, z, np.arange(self.n)
        self._x, self._y, self._z, self.src = _f8(ax), _f8(ay), _f8(az), src  # must outlive the handle
        st = ctypes.c_int(0)
        self._h = lib().sph_oracle_tree_new(self._x.shape[0], _ptr(self._x), _ptr(self._y), _ptr(self._z),
                                            ctypes.byref(st))
        if not self._h:
            raise ValueError(f"oracle tree build failed with status {st.value}")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().sph_oracle_tree_free(self._h)
            self._h = None

    def density_pass(self, mass, h0, k: int, targets, max_iterations: int = 100, threads: int = 0) -> OracleResult:
        m = _f8(mass)[self.src]
        h = _f8(h0)[self.src].copy()
        na = h.shape[0]
        rho = np.zeros(na, dtype=np.float64)
        flags = np.zeros(na, dtype=np.uint8)
        todo = np.zeros(max(max_iterations, 1) + 1, dtype=np.int64)
        info = np.zeros(4, dtype=np.int64)
        tg = np.ascontiguousarray(targets, dtype=np.int64)
        st = lib().sph_oracle_density_pass_tree(self._h, _ptr(m), _ptr(h), _ptr(rho), _ptr(flags), k,
                                                max_iterations, threads, _ptr(tg), tg.shape[0], _ptr(todo),
                                                todo.shape[0], _ptr(info))
        if st:
            raise ValueError(f"oracle density pass failed with status {st}")
        it = int(info[0])
        return OracleResult(h[:self.n], rho[:self.n], flags[:self.n], todo[:it].copy(), it, int(info[3]))


def kernel_w(r, h):
    return float(lib().sph_oracle_w(float(r), float(h)))


# ---------------------------------------------------------------------------
# numpy helpers
# ---------------------------------------------------------------------------

def brute_force(x, y, z, mass, k: int):
    """All-pairs h (K-th other-particle distance) and density, small N only.

    Mirrors the reference test oracle (test_density.py:33-46): h from the
    sorted distances, density summed over every particle inside the support.
    """
    pos = np.column_stack([_f8(x), _f8(y), _f8(z)])
    m = _f8(mass)
    n = pos.shape[0]
    diff = pos[None, :, :] - pos[:, None, :]
    d2 = (diff[..., 0] * diff[..., 0] + diff[..., 1] * diff[..., 1]) + diff[..., 2] * diff[..., 2]
    h = np.empty(n)
    rho = np.empty(n)
    for i in range(n):
        others = np.sort(np.delete(d2[i], i))
        h[i] = math.sqrt(others[k - 1])
        r = np.sqrt(d2[i])
        q = r / h[i]
        u = 1.0 - q
        u4 = (u * u) ** 2
        w = np.where(q < 1.0, WENDLAND_C6_NORM / (h[i] ** 3) * u4 * u4 *
                     (1.0 + q * (8.0 + q * (25.0 + 32.0 * q))), 0.0)
        rho[i] = float(np.sum(m * w))
    return h, rho


def periodic_images(x, y, z, box: float, margin: float):
    """Originals followed by every periodic image within ``margin`` of the
    box (26 shifts).  Image coordinates are ``x + s*box`` rounded in fp64,
    which is exactly what the GPU periodic mode computes.  Returns
    (x, y, z, source index)."""
    x, y, z = _f8(x), _f8(y), _f8(z)
    xs, ys, zs, src = [x], [y], [z], [np.arange(x.shape[0])]
    for sx in (-1, 0, 1):
        for sy in (-1, 0, 1):
            for sz in (-1, 0, 1):
                if sx == sy == sz == 0:
                    continue
                ix = x + sx * box
                iy = y + sy * box
                iz = z + sz * box
                keep = ((ix >= -margin) & (ix < box + margin) & (iy >= -margin) &
                        (iy < box + margin) & (iz >= -margin) & (iz < box + margin))
                xs.append(ix[keep]); ys.append(iy[keep]); zs.append(iz[keep])
                src.append(np.nonzero(keep)[0])
    return (np.concatenate(xs), np.concatenate(ys), np.concatenate(zs),
            np.concatenate(src))


def periodic_crop(x, y, z, box: float, targets, margin: float) -> np.ndarray:
    """Sorted indices of every particle whose minimum-image Chebyshev distance
    to some target is at most ``margin`` (a superset: whole grid cells of side
    >= margin around each target's cell, wrapped).  Each target's h and rho
    depend only on the particles within its h (reference density.py:11-13),
    so the periodic oracle over the crop, with every target's search radius
    below ``margin``, gives the full set's answer for the targets; the crop
    keeps the originals' relative order, so (d2, index) ties break alike."""
    ncell = int(box // margin)
    if ncell < 3:
        return np.arange(np.asarray(x).shape[0])
    cell = box / ncell
    tg = np.asarray(targets)

    def cid(ax, ay, az):
        ix = np.minimum((np.asarray(ax) / cell).astype(np.int64), ncell - 1)
        iy = np.minimum((np.asarray(ay) / cell).astype(np.int64), ncell - 1)
        iz = np.minimum((np.asarray(az) / cell).astype(np.int64), ncell - 1)
        return ix, iy, iz

    tx, ty, tz = cid(np.asarray(x)[tg], np.asarray(y)[tg], np.asarray(z)[tg])
    need = set()
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                c = (((tx + dx) % ncell) * ncell + (ty + dy) % ncell) * ncell + (tz + dz) % ncell
                need.update(c.tolist())
    need = np.array(sorted(need), dtype=np.int64)
    keep = np.zeros(x.shape[0], dtype=bool)
    step = 1 << 24
    for a in range(0, x.shape[0], step):
        ix, iy, iz = cid(x[a:a + step], y[a:a + step], z[a:a + step])
        keep[a:a + step] = np.isin((ix * ncell + iy) * ncell + iz, need)
    return np.nonzero(keep)[0]


def density_pass_periodic(x, y, z, mass, h0, k: int, box: float,
                          max_iterations: int = 100, threads: int = 0,
                          margin: float | None = None, targets=None) -> OracleResult:
    """Periodic-box pass via image augmentation: the open-boundary reference
    algorithm run on the originals plus images within ``margin`` of the box;
    results of the first N (the originals) are returned.  The margin doubles
    until it exceeds every converged h of the originals."""
    n = np.asarray(x).shape[0]
    if margin is None:
        margin = min(0.5 * box, 2.0 * float(np.max(np.abs(h0))) if n else box)
    while True:
        ax, ay, az, src = periodic_images(x, y, z, box, margin)
        am = _f8(mass)[src]
        ah = _f8(h0)[src]
        tg = np.arange(n) if targets is None else np.asarray(targets)
        res = density_pass(ax, ay, az, am, ah, k, max_iterations, threads, targets=tg)
        hmax = float(np.max(res.h[tg])) if tg.size else 0.0
        if hmax < margin or margin >= box:
            res.h = res.h[:n]
            res.rho = res.rho[:n]
            res.flags = res.flags[:n]
            return res
        margin = min(2.0 * margin, box)
