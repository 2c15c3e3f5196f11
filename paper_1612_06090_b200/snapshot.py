"""SPHK snapshots (the reference's checksummed workload files, snapshot.py:1-21
of sphlab) read straight into device memory.

Format (little-endian): magic "SPHK", u32 version (1), u32 section count,
then per section: u32 name length, name (UTF-8), u64 payload length, payload,
u64 FNV-1a-64 of the payload.  A "particles" payload is u64 n followed by the
live fields one after the other, each as n values of its own width: id i8,
x y z mass smoothing_length density f8, needs_recompute u1
(particles.py:20-29, snapshot.py:173-184) — already structure-of-arrays.

``load_particles_device`` maps the file, copies x, y, z, mass and
smoothing_length from the mapped payload into device tensors through pinned
staging, and verifies every section checksum (native FNV-1a, the library's
``sph_fnv1a64``) on a host thread concurrently with the copies; nothing is
returned before every checksum has passed (the reference's guarantee,
snapshot.py:11-15).  Error types mirror the reference's.
"""

from __future__ import annotations

import json
import mmap
import struct
import threading

import numpy as np

MAGIC = b"SPHK"
VERSION = 1
LIVE_FIELDS = [("id", "<i8"), ("x", "<f8"), ("y", "<f8"), ("z", "<f8"), ("mass", "<f8"),
               ("smoothing_length", "<f8"), ("density", "<f8"), ("needs_recompute", "u1")]


class SnapshotError(Exception):
    """Base for everything that can go wrong with snapshot files."""


class SnapshotIOError(SnapshotError):
    pass


class BadMagicError(SnapshotError):
    pass


class VersionError(SnapshotError):
    pass


class TruncatedError(SnapshotError):
    pass


class ChecksumError(SnapshotError):
    def __init__(self, section: str, stored: int, computed: int):
        self.section = section
        super().__init__(f"section {section!r}: stored checksum {stored:#018x} != computed {computed:#018x}")


def checksum64(data) -> int:
    """FNV-1a 64 of a byte buffer (native, the library's sph_fnv1a64)."""
    from . import _lib
    return _lib.fnv1a64_native(np.frombuffer(memoryview(data), dtype=np.uint8))


def dump(path, sections) -> None:
    """Write named byte blocks in mapping order (the reference's layout)."""
    parts = [MAGIC, struct.pack("<II", VERSION, len(sections))]
    for name, payload in sections.items():
        raw = bytes(payload)
        nb = name.encode("utf-8")
        parts += [struct.pack("<I", len(nb)), nb, struct.pack("<Q", len(raw)), raw,
                  struct.pack("<Q", checksum64(raw))]
    try:
        with open(path, "wb") as f:
            f.write(b"".join(parts))
    except OSError as exc:
        raise SnapshotIOError(f"cannot write snapshot {path!r}: {exc}") from exc


def encode_particles(fields: dict) -> bytes:
    """Field-by-field encoding of a particle set given as arrays (or a record
    array with the reference's field names)."""
    names = fields.dtype.names if getattr(fields, "dtype", None) is not None else tuple(fields.keys())
    n = len(fields["x"])
    parts = [struct.pack("<Q", n)]
    for name, dt in LIVE_FIELDS:
        if name in names:
            v = np.asarray(fields[name])
        else:  # fields the caller does not have: ids 0..n-1, zeros
            v = np.arange(n) if name == "id" else np.zeros(n)
        parts.append(np.ascontiguousarray(v).astype(np.dtype(dt), copy=False).tobytes())
    return b"".join(parts)


class _Sections:
    """Section table of a mapped file: name -> (offset, length, stored checksum)."""

    def __init__(self, path):
        self.path = path
        try:
            self.f = open(path, "rb")
            self.mm = mmap.mmap(self.f.fileno(), 0, access=mmap.ACCESS_READ) if self._size() else b""
        except OSError as exc:
            raise SnapshotIOError(f"cannot read snapshot {path!r}: {exc}") from exc
        self.table = {}
        off = 0
        magic = self._take(off, 4, "magic")
        if magic != MAGIC:
            raise BadMagicError(f"snapshot {path!r}: bad magic {magic!r}, expected {MAGIC!r}")
        off = 4
        version = struct.unpack("<I", self._take(off, 4, "version"))[0]
        if version != VERSION:
            raise VersionError(f"snapshot {path!r}: unsupported version {version}, expected {VERSION}")
        count = struct.unpack("<I", self._take(off + 4, 4, "section count"))[0]
        off += 8
        for _ in range(count):
            nl = struct.unpack("<I", self._take(off, 4, "section name length"))[0]
            name = bytes(self._take(off + 4, nl, "section name")).decode("utf-8")
            off += 4 + nl
            plen = struct.unpack("<Q", self._take(off, 8, f"payload length of {name!r}"))[0]
            self._take(off + 8, plen, f"payload of {name!r}")
            stored = struct.unpack("<Q", self._take(off + 8 + plen, 8, f"checksum of {name!r}"))[0]
            self.table[name] = (off + 8, plen, stored)
            off += 16 + plen

    def _size(self):
        import os
        return os.fstat(self.f.fileno()).st_size

    def _take(self, off, n, what):
        if off + n > len(self.mm):
            raise TruncatedError(f"snapshot {self.path!r} truncated while reading {what} (need {n} bytes at "
                                 f"offset {off}, have {len(self.mm) - off})")
        return memoryview(self.mm)[off:off + n]

    def payload(self, name):
        off, n, _ = self.table[name]
        return memoryview(self.mm)[off:off + n]

    def verify(self):
        for name, (off, n, stored) in self.table.items():
            got = checksum64(memoryview(self.mm)[off:off + n])
            if got != stored:
                raise ChecksumError(name, stored, got)

    def close(self):
        if isinstance(self.mm, mmap.mmap):
            try:
                self.mm.close()
            except BufferError:  # numpy views still alive: the mapping goes with them
                pass
        self.f.close()


def load(path) -> dict:
    """name -> bytes, every checksum verified (reference snapshot.load)."""
    s = _Sections(path)
    try:
        s.verify()
        return {name: bytes(s.payload(name)) for name in s.table}
    finally:
        s.close()


def _field_views(payload, what):
    if len(payload) < 8:
        raise TruncatedError("particle payload shorter than its count header")
    n = struct.unpack("<Q", bytes(payload[:8]))[0]
    off = 8
    views = {}
    for name, dt in LIVE_FIELDS:
        d = np.dtype(dt)
        nb = n * d.itemsize
        if off + nb > len(payload):
            raise TruncatedError(f"particle payload truncated in field {name!r}")
        views[name] = np.frombuffer(payload, dtype=d, count=n, offset=off)
        off += nb
    if off != len(payload):
        raise SnapshotError(f"particle payload has {len(payload) - off} trailing bytes")
    return n, views


def decode_particles(payload) -> dict:
    """Host arrays of the live fields of a particles payload."""
    n, views = _field_views(memoryview(payload), "particles")
    return {k: v.copy() for k, v in views.items()}


def load_particles_device(path, device: int = 0, fields=("x", "y", "z", "mass", "smoothing_length"),
                          section: str = "particles", chunk_bytes: int = 64 << 20):
    """The snapshot's particle fields as float64 device tensors (plus the
    "meta" section parsed when present).  The copies run while a host thread
    verifies the checksums; a checksum failure raises before returning."""
    import torch
    s = _Sections(path)
    try:
        if section not in s.table:
            raise SnapshotError(f"{path!r} has no {section!r} section")
        err = []

        def check():
            try:
                s.verify()
            except SnapshotError as e:
                err.append(e)

        th = threading.Thread(target=check)
        th.start()
        n, views = _field_views(s.payload(section), section)
        dev = torch.device("cuda", device)
        out = {}
        stage = torch.empty(max(1, min(chunk_bytes, n * 8)), dtype=torch.uint8).pin_memory()
        for name in fields:
            v = views[name]
            t = torch.empty(n, dtype=torch.float64, device=dev)
            tb = t.view(torch.uint8)
            src = v.view(np.uint8)
            for o in range(0, src.size, stage.numel()):
                m = min(stage.numel(), src.size - o)
                stage[:m].numpy()[:] = src[o:o + m]
                tb[o:o + m].copy_(stage[:m], non_blocking=False)
            out[name] = t
        meta = json.loads(bytes(s.payload("meta"))) if "meta" in s.table else {}
        th.join()
        if err:
            raise err[0]
        return out, meta
    finally:
        s.close()


def density_pass_snapshot(path, k: int | None = None, device: int = 0, max_iterations: int = 100):
    """`sphlab run` for one snapshot on the GPU: particles streamed to the
    device, the pass on device-resident arrays; returns host (h, rho, flags,
    PassStats) in the snapshot's particle order."""
    import ctypes

    import torch

    from . import _lib
    from .density import DEFAULT_K, _raise_for, _stats_from, initial_smoothing_length

    f, meta = load_particles_device(path, device)
    n = f["x"].numel()
    L = _lib.load()
    ctx = _lib.context(device)
    h = f["smoothing_length"].clone()
    # the reference CLI (cli.py:159-163): K defaults to the snapshot's
    # k_neighbors, else DEFAULT_K; an explicit K that differs from it resets
    # every h0 to initial_smoothing_length(box_side, n, K)
    if k is not None and k != meta.get("k_neighbors"):
        h.fill_(initial_smoothing_length(float(meta.get("box_side", 1.0)), n, int(k)))
    k = int(k if k is not None else meta.get("k_neighbors", DEFAULT_K))
    rho = torch.empty(n, dtype=torch.float64, device=h.device)
    flags = torch.empty(n, dtype=torch.uint8, device=h.device)
    prm = _lib.SphParams(n=n, k=k, max_iterations=max_iterations, precision=_lib.PRECISION["auto"], periodic=0,
                         box=0.0, kernel=0, reserved=0, n_targets=0)
    st = _lib.SphStats()
    torch.cuda.synchronize(h.device)
    vp = ctypes.c_void_p
    rc = L.sph_density_pass_device(ctx, prm, vp(f["x"].data_ptr()), vp(f["y"].data_ptr()), vp(f["z"].data_ptr()),
                                   vp(f["mass"].data_ptr()), vp(h.data_ptr()), vp(rho.data_ptr()),
                                   vp(flags.data_ptr()), st)
    _raise_for(rc, ctx)
    return h.cpu().numpy(), rho.cpu().numpy(), flags.cpu().numpy(), _stats_from(st, 0.0)
