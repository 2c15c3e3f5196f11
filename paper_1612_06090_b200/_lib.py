"""ctypes binding of libsph_b200.so (the C ABI declared in include/sph_b200.h).

This module is the reference-side stub INTEGRATION.md describes: plain
pointers and sizes, no torch types.  The library is built in-tree by
``__graft_entry__.build()`` (or ``make -C paper_1612_06090_b200``).  There is
no CPU fallback: if the library or a CUDA device is missing, every compute
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsph_b200.so")

SPH_OK, SPH_NOT_CONVERGED, SPH_DEGENERATE, SPH_INVALID, SPH_CUDA_ERROR, SPH_UNSUPPORTED = range(6)
PRECISION = {"f64": 0, "f32": 1, "auto": 2}
KERNELS = {"wendland_c6": 0, "m4": 1}
MAX_TODO = 128

EXPORTED_SYMBOLS = (
    "sph_ctx_create", "sph_ctx_destroy", "sph_last_error", "sph_device_count",
    "sph_density_pass", "sph_density_pass_device", "sph_sort_perm",
    "sph_neighbor_counts", "sph_fnv1a64", "sph_ctx_stream", "sph_fp32_peak", "sph_uniform_box_device",
    "sph_morton_keys_device", "sph_decomp_pack_rows_device", "sph_decomp_gather_rows_device",
    "sph_decomp_row_keys_device", "sph_decomp_level_bounds_device", "sph_decomp_window_bounds_device",
    "sph_decomp_ghost_mask_device", "sph_decomp_group_boxes_device", "sph_bbox_device", "sph_range_query",
    "sph_nfw_positions_device", "sph_density_pass_multi", "sph_octree_build", "sph_octree_query",
    "sph_sort_perm_ex",
)


class SphParams(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("k", ctypes.c_int32), ("max_iterations", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("periodic", ctypes.c_int32), ("box", ctypes.c_double),
                ("kernel", ctypes.c_int32), ("reserved", ctypes.c_int32), ("n_targets", ctypes.c_int64)]


class SphStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("n_todo", ctypes.c_int32),
                ("todo_sizes", ctypes.c_int64 * MAX_TODO), ("t_stage_ms", ctypes.c_double * 8),
                ("pair_tests", ctypes.c_int64), ("accepted_pairs", ctypes.c_int64),
                ("search_pair_tests", ctypes.c_int64), ("bad_index", ctypes.c_int64),
                ("unconverged", ctypes.c_int64), ("gpu_launches", ctypes.c_int32),
                ("search_rounds", ctypes.c_int32), ("select_rounds", ctypes.c_int32),
                ("n_nodes", ctypes.c_int32), ("t_kernel_ms", ctypes.c_double * 4),
                ("t_known_ms", ctypes.c_double), ("known_fallbacks", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {
            "iterations": self.iterations,
            "todo_sizes": [int(self.todo_sizes[i]) for i in range(min(self.n_todo, MAX_TODO))],
            "t_stage_ms": {name: float(self.t_stage_ms[i]) for i, name in enumerate(
                ("h2d", "tree", "search", "select", "density", "finalize", "d2h", "total"))},
            "pair_tests": int(self.pair_tests),
            "accepted_pairs": int(self.accepted_pairs),
            "search_pair_tests": int(self.search_pair_tests),
            "bad_index": int(self.bad_index),
            "unconverged": int(self.unconverged),
            "gpu_launches": int(self.gpu_launches),
            "search_rounds": int(self.search_rounds),
            "select_rounds": int(self.select_rounds),
            "n_nodes": int(self.n_nodes),
            "t_kernel_ms": {name: float(self.t_kernel_ms[i]) for i, name in enumerate(
                ("search", "select", "density", "tree"))},
            "t_known_ms": float(self.t_known_ms),
            "known_fallbacks": int(self.known_fallbacks),
        }


_lib = None
_lock = threading.Lock()
_ctx = {}


def load():
    """Load the native library (raises OSError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        L.sph_ctx_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
        L.sph_ctx_destroy.argtypes = [vp]
        L.sph_last_error.argtypes = [vp]
        L.sph_last_error.restype = ctypes.c_char_p
        L.sph_device_count.restype = ctypes.c_int
        L.sph_density_pass.argtypes = [vp, ctypes.POINTER(SphParams), vp, vp, vp, i64, vp, i64, vp, i64,
                                       vp, i64, vp, i64, ctypes.POINTER(SphStats)]
        L.sph_density_pass_device.argtypes = [vp, ctypes.POINTER(SphParams), vp, vp, vp, vp, vp, vp, vp,
                                              ctypes.POINTER(SphStats)]
        L.sph_sort_perm_ex.argtypes = [vp, i32, i64, vp, vp, vp, i32, vp]
        L.sph_octree_build.argtypes = [vp, i32, i64, vp, vp, vp]
        L.sph_octree_query.argtypes = [vp, i64, vp, vp, vp, i64, vp, vp, vp, ctypes.POINTER(ctypes.c_int64)]
        L.sph_density_pass_multi.argtypes = [ctypes.POINTER(vp), i32, ctypes.POINTER(SphParams), vp, vp, vp, i64,
                                             vp, i64, vp, i64, vp, i64, vp, i64, ctypes.POINTER(SphStats)]
        L.sph_sort_perm.argtypes = [vp, i32, i64, vp, vp, vp, vp]
        L.sph_neighbor_counts.argtypes = [vp, i32, i32, ctypes.c_double, i64, vp, vp, vp, vp, vp,
                                          ctypes.POINTER(SphStats)]
        L.sph_fp32_peak.argtypes = [vp]
        L.sph_fp32_peak.restype = ctypes.c_double
        L.sph_ctx_stream.argtypes = [vp]
        L.sph_ctx_stream.restype = vp
        L.sph_fnv1a64.argtypes = [vp, ctypes.c_size_t]
        L.sph_fnv1a64.restype = ctypes.c_uint64
        L.sph_uniform_box_device.argtypes = [vp, i64, ctypes.c_uint64, ctypes.c_double, vp, vp, vp]
        L.sph_nfw_positions_device.argtypes = [vp, i64, i64, vp, vp, ctypes.c_double, ctypes.c_double,
                                               ctypes.c_uint64, ctypes.c_double, vp, vp, vp, vp]
        L.sph_morton_keys_device.argtypes = [vp, i32, i64, vp, vp, vp, ctypes.POINTER(ctypes.c_double),
                                             ctypes.c_double, vp]
        L.sph_decomp_pack_rows_device.argtypes = [vp, i32, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.sph_decomp_gather_rows_device.argtypes = [vp, i64, i32, vp, vp, vp]
        L.sph_decomp_row_keys_device.argtypes = [vp, i64, vp, vp]
        L.sph_decomp_level_bounds_device.argtypes = [vp, i64, i32, vp, ctypes.c_double, vp]
        L.sph_decomp_window_bounds_device.argtypes = [vp, i64, i32, i32, vp, ctypes.c_double, vp]
        L.sph_bbox_device.argtypes = [vp, i32, i64, vp, vp, vp, vp]
        L.sph_range_query.argtypes = [vp, i32, i64, vp, vp, vp, vp, vp, vp, vp]
        L.sph_decomp_ghost_mask_device.argtypes = [vp, i64, vp, vp, vp, i32, vp, i64, vp, vp, i32, ctypes.c_double,
                                                   vp]
        L.sph_decomp_group_boxes_device.argtypes = [vp, i64, vp, vp, i32, vp, vp, vp]
        _lib = L
        return L


def fnv1a64_native(buf: np.ndarray) -> int:
    L = load()
    b = np.ascontiguousarray(buf, dtype=np.uint8)
    return int(L.sph_fnv1a64(b.ctypes.data_as(ctypes.c_void_p), b.nbytes))


def device_count() -> int:
    return int(load().sph_device_count())


def context(device: int = 0):
    """Per-device context (stream + device buffers reused across calls)."""
    L = load()
    with _lock:
        c = _ctx.get(device)
        if c is None:
            if L.sph_device_count() <= 0:
                raise RuntimeError("no CUDA device visible: the B200 pass has no CPU fallback")
            h = ctypes.c_void_p()
            rc = L.sph_ctx_create(ctypes.byref(h), device)
            if rc != SPH_OK:
                raise RuntimeError(f"sph_ctx_create(device={device}) failed with status {rc}")
            c = h
            _ctx[device] = c
        return c


def drop_context(device: int = 0) -> None:
    """Destroy the cached per-device context (frees its device buffers; the
    next call on the device creates a fresh one)."""
    with _lock:
        c = _ctx.pop(device, None)
    if c is not None:
        load().sph_ctx_destroy(c)


def new_context(device: int = 0):
    """A private context (its own stream and buffers), e.g. one per in-process
    rank of an emulated decomposition; never destroyed before exit."""
    L = load()
    if L.sph_device_count() <= 0:
        raise RuntimeError("no CUDA device visible: the B200 pass has no CPU fallback")
    h = ctypes.c_void_p()
    rc = L.sph_ctx_create(ctypes.byref(h), device)
    if rc != SPH_OK:
        raise RuntimeError(f"sph_ctx_create(device={device}) failed with status {rc}")
    with _lock:
        _private.append(h)
    return h


_private = []
_multi = {}


def contexts(devices) -> list:
    """One distinct context per entry of ``devices`` (a multi-device pass;
    the same device may repeat, each repeat then gets its own private
    context and stream, so the split is exercised on one GPU too)."""
    out, seen = [], {}
    for d in devices:
        d = int(d)
        i = seen.get(d, 0)
        seen[d] = i + 1
        if i == 0:
            out.append(context(d))
        else:
            with _lock:
                c = _multi.get((d, i))
            if c is None:
                c = new_context(d)
                with _lock:
                    _multi[(d, i)] = c
            out.append(c)
    return out


def stream_handle(ctx) -> int:
    """The context's cudaStream_t (for torch.cuda.ExternalStream)."""
    return int(load().sph_ctx_stream(ctx) or 0)


def last_error(ctx) -> str:
    msg = load().sph_last_error(ctx)
    return msg.decode() if msg else ""


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)
