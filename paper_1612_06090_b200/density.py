"""The drop-in density pass: the reference's operator API on the B200 path.

Mirrors ``sphlab.density`` (density.py of the reference): the same names,
argument meaning, return values and error behaviour, with the work done by
``libsph_b200.so``.  ``compute_density_pass`` reads x, y, z, mass and the
initial smoothing_length straight out of the caller's packed records (the
C ABI takes base pointer + record stride), and writes smoothing_length,
density and needs_recompute back into them, exactly like the reference
(density.py:286-413).

What the GPU computes is the reference's converged state, not its
iteration path: h_i is the exact fp64 distance to the K-th nearest other
particle (the reference's fixed point, density.py:11-13) and rho_i the
Wendland C6 sum over the particles inside it.  The reference's growth-only
todo trace (``PassStats.todo_sizes``) is a pure function of h0 and that
distance, so the library reproduces it exactly (see k_finalize in
csrc/sph_api.cu) without running the CPU's rounds.

The variant lattice (scheduler / layout / loop style / selector) only
changes how the reference's CPU threads get there; every preset gives the
same numbers (density.py:11-18), so the GPU pass accepts any config and
uses only ``k_neighbors``.  ``thread_count`` is validated and otherwise
ignored (GPU work is scheduled on the device).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .particles import DEFAULT_AOS_RECORD_BYTES, LayoutKind, is_packed_record_array

DEFAULT_K = 295
H_GROWTH = 2.0 ** (1.0 / 3.0)
DEFAULT_MAX_ITERATIONS = 100
DEFAULT_CHUNK_SIZE = 16
PHASE_NAMES = ("tree_build", "search", "select", "interact", "layout")


class SchedulerKind(Enum):
    LOCKED_QUEUE = "locked-queue"
    TODO_LIST = "todo-list"
    DYNAMIC_FOR = "dynamic-for"


class LoopStyle(Enum):
    BRANCHY = "branchy"
    BRANCH_LOWERED = "branch-lowered"


class SelectorKind(Enum):
    FULL_SORT = "full-sort"
    QUICK_SELECT = "quick-select"


class ConvergenceError(RuntimeError):
    """The todo list failed to empty within the iteration budget."""


class DegenerateWorkloadError(RuntimeError):
    """A particle's K-th neighbor sits at zero distance (coincident cluster)."""


@dataclass(frozen=True)
class VariantConfig:
    scheduler_kind: SchedulerKind
    layout_kind: LayoutKind
    loop_style: LoopStyle
    selector_kind: SelectorKind
    k_neighbors: int = DEFAULT_K
    chunk_size: int = DEFAULT_CHUNK_SIZE

    def __post_init__(self):
        if self.k_neighbors < 1:
            raise ValueError(f"k_neighbors must be >= 1, got {self.k_neighbors}")
        if self.chunk_size < 1:
            raise ValueError(f"chunk_size must be >= 1, got {self.chunk_size}")

    def replace(self, **kw) -> "VariantConfig":
        from dataclasses import replace
        return replace(self, **kw)


PRESETS: dict[str, VariantConfig] = {
    "original": VariantConfig(SchedulerKind.LOCKED_QUEUE, LayoutKind.AOS, LoopStyle.BRANCHY,
                              SelectorKind.FULL_SORT),
    "todo-list": VariantConfig(SchedulerKind.TODO_LIST, LayoutKind.AOS, LoopStyle.BRANCHY,
                               SelectorKind.FULL_SORT),
    "lockless": VariantConfig(SchedulerKind.DYNAMIC_FOR, LayoutKind.AOS, LoopStyle.BRANCHY,
                              SelectorKind.FULL_SORT),
    "soa": VariantConfig(SchedulerKind.DYNAMIC_FOR, LayoutKind.SOA, LoopStyle.BRANCHY,
                         SelectorKind.FULL_SORT),
    "vectorised": VariantConfig(SchedulerKind.DYNAMIC_FOR, LayoutKind.SOA, LoopStyle.BRANCH_LOWERED,
                                SelectorKind.FULL_SORT),
    "optimised": VariantConfig(SchedulerKind.DYNAMIC_FOR, LayoutKind.SOA, LoopStyle.BRANCH_LOWERED,
                               SelectorKind.QUICK_SELECT),
}


def preset_config(name: str, **overrides) -> VariantConfig:
    try:
        cfg = PRESETS[name]
    except KeyError:
        known = ", ".join(sorted(PRESETS))
        raise ValueError(f"unknown preset {name!r}; expected one of {known}")
    return cfg.replace(**overrides) if overrides else cfg


@dataclass
class PassStats:
    iteration_count: int
    todo_sizes: np.ndarray
    phase_times: dict[str, float]
    contention_time: float
    items_per_worker: np.ndarray  # shape (iterations, workers); one worker = the GPU
    skipped_items: int = 0
    t_total: float = 0.0
    device: dict = field(default_factory=dict)  # GPU counters (pair tests, stage times, launches)


def initial_smoothing_length(box_side: float, n_particles: int, k: int) -> float:
    """Radius enclosing k particles at uniform density (density.py:136-140)."""
    if n_particles < 1 or k < 1 or box_side <= 0.0:
        raise ValueError("need box_side > 0, n_particles >= 1, k >= 1")
    return box_side * (3.0 * k / (4.0 * math.pi * n_particles)) ** (1.0 / 3.0)


def adjust_smoothing_length(smoothing_length: float, found_count: int, k: int,
                            kth_distance: float | None = None) -> tuple[float, bool]:
    """One reference smoothing-length update step (density.py:143-157)."""
    if found_count < 0:
        raise ValueError(f"found_count must be >= 0, got {found_count}")
    if found_count < k:
        return smoothing_length * H_GROWTH, True
    if kth_distance is None:
        raise ValueError("kth_distance is required when found_count >= k")
    return float(kth_distance), False


def density_interact(masses: np.ndarray, smoothing_length: float, neighbor_dist2: np.ndarray,
                     neighbor_index: np.ndarray, loop_style: LoopStyle = LoopStyle.BRANCHY) -> float:
    """Sum m_j W(r_ij, h) over a candidate list in list order (density.py:174-190).

    A host-side helper of the reference API (single-shot, not the pass).
    """
    d2 = np.ascontiguousarray(neighbor_dist2, dtype=np.float64)
    idx = np.ascontiguousarray(neighbor_index, dtype=np.int64)
    if d2.shape != idx.shape or d2.ndim != 1:
        raise ValueError("neighbor arrays must be 1-D and of equal length")
    m = np.ascontiguousarray(masses, dtype=np.float64)
    h = float(smoothing_length)
    norm = 1365.0 / (64.0 * math.pi) / (h * h * h)
    rho = 0.0
    h2 = h * h
    for n in range(d2.shape[0]):
        if loop_style is LoopStyle.BRANCHY and not d2[n] < h2:
            continue
        q = math.sqrt(d2[n]) / h
        if q < 1.0:
            u = 1.0 - q
            u2 = u * u
            u4 = u2 * u2
            rho += m[idx[n]] * (norm * (u4 * u4 * (1.0 + q * (8.0 + q * (25.0 + 32.0 * q)))))
    return float(rho)


def _raise_for(rc: int, ctx) -> None:
    if rc == _lib.SPH_OK:
        return
    msg = _lib.last_error(ctx)
    if rc == _lib.SPH_NOT_CONVERGED:
        raise ConvergenceError(msg)
    if rc == _lib.SPH_DEGENERATE:
        raise DegenerateWorkloadError(msg)
    if rc == _lib.SPH_INVALID:
        raise ValueError(msg)
    raise RuntimeError(msg or f"sph library status {rc}")


def _stats_from(st: _lib.SphStats, t_total: float) -> PassStats:
    d = st.as_dict()
    todo = np.array(d["todo_sizes"], dtype=np.int64)
    ts = d["t_stage_ms"]
    tk = d["t_kernel_ms"]
    phase = {
        "tree_build": ts["tree"] / 1e3,
        "search": ts["search"] / 1e3,
        "select": ts["select"] / 1e3,
        "interact": ts["density"] / 1e3,
        "layout": (ts["h2d"] + ts["finalize"] + ts["d2h"]) / 1e3,
    }
    return PassStats(iteration_count=int(st.iterations), todo_sizes=todo, phase_times=phase,
                     contention_time=0.0, items_per_worker=todo.reshape(-1, 1).copy(),
                     skipped_items=0, t_total=t_total, device=d)


def _multi_stats(sts, t_total: float) -> PassStats:
    """PassStats of a multi-device pass: the merged trace, items_per_worker =
    each device's own todo trace (iterations x devices, density.py:407-409)."""
    merged = _stats_from(sts[-1], t_total)
    iters = merged.iteration_count
    per = np.zeros((len(merged.todo_sizes), len(sts) - 1), dtype=np.int64)
    for d, st in enumerate(sts[:-1]):
        t = np.array(st.todo_sizes[:min(st.iterations, _lib.MAX_TODO)], dtype=np.int64)
        per[:t.size, d] = t
    merged.items_per_worker = per[:max(iters, 0)] if iters else per[:0]
    merged.device = dict(merged.device, per_device=[_lib.SphStats.as_dict(s) for s in sts[:-1]])
    return merged


def _run_multi(devices, prm, x, y, z, pos_stride, m, m_stride, h, h_stride, rho, rho_stride, flags, f_stride):
    import ctypes
    L = _lib.load()
    ctxs = _lib.contexts(devices)
    arr = (ctypes.c_void_p * len(ctxs))(*[c.value if hasattr(c, "value") else c for c in ctxs])
    sts = (_lib.SphStats * (len(ctxs) + 1))()
    rc = L.sph_density_pass_multi(arr, len(ctxs), prm, x, y, z, pos_stride, m, m_stride, h, h_stride, rho,
                                  rho_stride, flags, f_stride, sts)
    return rc, ctxs[0], list(sts)


def compute_density_pass(particles: np.ndarray, config: VariantConfig, thread_count: int = 1,
                         max_iterations: int = DEFAULT_MAX_ITERATIONS, *, precision: str = "auto",
                         periodic: bool = False, box: float | None = None,
                         kernel: str = "wendland_c6", device: int = 0,
                         devices=None) -> tuple[np.ndarray, PassStats]:
    """Run the density pass on the GPU over the caller's particle records.

    Same contract as the reference (density.py:286-413): reads positions,
    masses and the initial smoothing_length; writes smoothing_length,
    density and needs_recompute back; returns (a new float64 density array,
    PassStats).  Raises ValueError / ConvergenceError /
    DegenerateWorkloadError like the reference.

    Extensions (keyword-only): ``precision`` "auto" (fp32 kernels when every
    coordinate is fp32-representable, results still bit-exact against the
    fp64 reference), "f64" or "f32"; ``periodic``/``box`` for a periodic
    cube [0, box)^3 (the reference has open boundaries only); ``kernel``
    "wendland_c6" (the reference) or "m4"; ``devices`` (a list of device
    ids, repeats allowed) splits the targets over several GPUs
    (sph_density_pass_multi): PassStats.items_per_worker then has one column
    per device, as the reference's has one per worker thread.
    """
    n = particles.shape[0]
    if n == 0:
        raise ValueError("workload must contain at least one particle")
    if thread_count < 1:
        raise ValueError(f"thread_count must be >= 1, got {thread_count}")
    if precision not in ("auto", "f64"):
        if precision != "f32":
            raise ValueError(f"unknown precision {precision!r}")
    if periodic and (box is None or not box > 0.0):
        raise ValueError("periodic mode needs box > 0")
    t0 = time.perf_counter()
    multi = devices is not None and len(devices) > 1
    ctx = _lib.context(devices[0] if devices else device)
    L = _lib.load()

    prm = _lib.SphParams(n=n, k=config.k_neighbors, max_iterations=max_iterations,
                         precision=_lib.PRECISION["auto" if precision == "f32" else precision],
                         periodic=1 if periodic else 0, box=float(box or 0.0),
                         kernel=_lib.KERNELS[kernel], reserved=0)
    st = _lib.SphStats()
    packed = (is_packed_record_array(particles) and particles.ndim == 1
              and particles.flags["C_CONTIGUOUS"] and particles.flags["WRITEABLE"])
    if packed:
        base = particles.ctypes.data
        stride = particles.dtype.itemsize
        vp = ctypes_addr
        if multi:
            rc, ctx, sts = _run_multi(devices, prm, vp(base + 8), vp(base + 16), vp(base + 24), stride,
                                      vp(base + 32), stride, vp(base + 40), stride, vp(base + 48), stride,
                                      vp(base + 56), stride)
        else:
            rc = L.sph_density_pass(ctx, prm, vp(base + 8), vp(base + 16), vp(base + 24), stride,
                                    vp(base + 32), stride, vp(base + 40), stride, vp(base + 48), stride,
                                    vp(base + 56), stride, st)
    else:
        x = np.ascontiguousarray(particles["x"], dtype=np.float64)
        y = np.ascontiguousarray(particles["y"], dtype=np.float64)
        z = np.ascontiguousarray(particles["z"], dtype=np.float64)
        m = np.ascontiguousarray(particles["mass"], dtype=np.float64)
        h = np.array(particles["smoothing_length"], dtype=np.float64)
        rho = np.zeros(n, dtype=np.float64)
        flags = np.zeros(n, dtype=np.uint8)
        if multi:
            rc, ctx, sts = _run_multi(devices, prm, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z), 8, _lib.ptr(m), 8,
                                      _lib.ptr(h), 8, _lib.ptr(rho), 8, _lib.ptr(flags), 1)
        else:
            rc = L.sph_density_pass(ctx, prm, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z), 8, _lib.ptr(m), 8,
                                    _lib.ptr(h), 8, _lib.ptr(rho), 8, _lib.ptr(flags), 1, st)
        if rc == _lib.SPH_OK:
            particles["smoothing_length"] = h
            particles["density"] = rho
            particles["needs_recompute"] = flags
    if rc != _lib.SPH_OK:
        particles["needs_recompute"] = 1
    _raise_for(rc, ctx)
    dt = time.perf_counter() - t0
    stats = _multi_stats(sts, dt) if multi else _stats_from(st, dt)
    return np.array(particles["density"], dtype=np.float64), stats


def ctypes_addr(a: int):
    import ctypes
    return ctypes.c_void_p(a)


def density_pass_soa(x, y, z, mass, h0, k: int, max_iterations: int = DEFAULT_MAX_ITERATIONS, *,
                     precision: str | None = None, periodic: bool = False, box: float = 0.0,
                     kernel: str = "wendland_c6", device: int = 0, out=None, n_targets: int | None = None,
                     devices=None):
    """SoA form of the pass on host arrays: returns (h, rho, flags, PassStats).

    ``precision`` defaults to the dtype of x ("f32" for float32 inputs).
    ``out`` = optional preallocated (h, rho, flags) host arrays (e.g. pinned);
    h is read as the initial smoothing length when ``h0`` is None.
    ``n_targets``: only particles [0, n_targets) are targets; the rest are
    ghosts (neighbour candidates only).  h0 / outputs then have n_targets
    entries.
    """
    x = np.ascontiguousarray(x)
    if precision is None:
        precision = "f32" if x.dtype == np.float32 else "f64"
    pdt = np.float32 if precision == "f32" else np.float64
    x = np.ascontiguousarray(x, dtype=pdt)
    y = np.ascontiguousarray(y, dtype=pdt)
    z = np.ascontiguousarray(z, dtype=pdt)
    m = np.ascontiguousarray(mass, dtype=np.float64)
    n = x.shape[0]
    if n == 0:
        raise ValueError("workload must contain at least one particle")
    nt = n if n_targets is None else int(n_targets)
    if not 0 < nt <= n:
        raise ValueError(f"n_targets must be in [1, {n}], got {nt}")
    if out is not None:
        h, rho, flags = out
        if h0 is not None:
            h[:] = h0
    else:
        h = np.array(np.broadcast_to(np.asarray(h0, dtype=np.float64), (nt,)))
        rho = np.zeros(nt, dtype=np.float64)
        flags = np.zeros(nt, dtype=np.uint8)
    multi = devices is not None and len(devices) > 1
    if multi and nt != n:
        raise ValueError("a multi-device pass takes every particle as a target (n_targets = None)")
    ctx = _lib.context(devices[0] if devices else device)
    L = _lib.load()
    prm = _lib.SphParams(n=n, k=k, max_iterations=max_iterations, precision=_lib.PRECISION[precision],
                         periodic=1 if periodic else 0, box=float(box), kernel=_lib.KERNELS[kernel],
                         reserved=0, n_targets=0 if nt == n else nt)
    st = _lib.SphStats()
    t0 = time.perf_counter()
    es = x.itemsize
    if multi:
        rc, ctx, sts = _run_multi(devices, prm, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z), es, _lib.ptr(m), 8,
                                  _lib.ptr(h), 8, _lib.ptr(rho), 8, _lib.ptr(flags), 1)
        _raise_for(rc, ctx)
        return h, rho, flags, _multi_stats(sts, time.perf_counter() - t0)
    rc = L.sph_density_pass(ctx, prm, _lib.ptr(x), _lib.ptr(y), _lib.ptr(z), es, _lib.ptr(m), 8,
                            _lib.ptr(h), 8, _lib.ptr(rho), 8, _lib.ptr(flags), 1, st)
    _raise_for(rc, ctx)
    return h, rho, flags, _stats_from(st, time.perf_counter() - t0)
