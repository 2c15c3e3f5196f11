"""Domain-decomposed density pass over P ranks (one process per GPU).

The reference runs on one shared-memory node (threads, scheduler.py of the
reference); it has no distributed mode.  Here each rank owns a contiguous
range of the same 63-bit x-major keys the ordering sorts by (the key of a
particle is its reference octree path, octree.py:93-104), so a rank's
particles form a compact piece of space, and the only data exchange of the
path is the ghost layer.  Everything stays in device memory; the collectives
are torch.distributed (NCCL over NVLink/NVSwitch on GPUs, gloo on CPU for the
tests), the per-rank compute is pluggable (``LibCompute``: libsph_b200 on the
rank's GPU; ``NumpyCompute``: any host pass, e.g. the CPU oracle in tests).

Steps of ``decomposed_pass`` (all ranks call it collectively):

  1. bbox all-reduce -> the common root cube (octree.py:324-328 arithmetic)
  2. keys from that cube (``sph_morton_keys_device``), count-balanced key
     splitters from all-gathered samples, one all-to-all moving each record
     (x, y, z, m, h0, global id, key) to its owner
  3. a guaranteed per-particle bound on h without any search: a particle in a
     level-l key cube that holds >= K+1 owned particles has K others within
     the cube's diagonal, so h <= sqrt(3) * side(l) for the deepest such l
     (a K-th neighbour among a subset is never nearer than among all)
  4. descriptors: owned particles grouped by a coarse key prefix, per group
     the tight box and the largest bound; all-gathered
  5. ghosts: every owned particle within a peer group's bound of that group's
     box (min-image when periodic) is sent to the peer (second all-to-all);
     a target's true neighbours all lie within its bound of its own box
  6. the final pass over owned + ghosts with the owned particles as targets
     (``sph_params.n_targets``): h is bit-identical to one GPU and so is the
     todo trace (a function of h0 and d2_K); densities agree to the fp32 sum
     order (bit-identical on the fp64 paths).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

KEY_LEVELS = 21
_SQRT3 = math.sqrt(3.0)


def root_cube(lo, hi):
    """Root centre and half-extent, fp64 op-for-op as octree.py:324-328."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    centre = 0.5 * (lo + hi)
    half = float(np.max(hi - lo)) * 0.5
    return centre, half


def morton_keys(pos: np.ndarray, centre: np.ndarray, half: float) -> np.ndarray:
    """63-bit x-major octant-path keys with the reference's centre arithmetic
    (the same keys the CUDA ordering computes, k_keys in csrc/sph_tree.cu)."""
    n = pos.shape[0]
    key = np.zeros(n, dtype=np.uint64)
    c = np.tile(np.asarray(centre, dtype=np.float64), (n, 1))
    h = float(half)
    for _ in range(KEY_LEVELS):
        b = pos >= c
        key = ((key << np.uint64(3)) | (b[:, 0].astype(np.uint64) << np.uint64(2))
               | (b[:, 1].astype(np.uint64) << np.uint64(1)) | b[:, 2].astype(np.uint64))
        h2 = h * 0.5
        c = np.where(b, c + h2, c - h2)
        h = h2
    return key


def box_distance2(pos: np.ndarray, lo: np.ndarray, hi: np.ndarray, periodic: bool, box: float) -> np.ndarray:
    """Squared distance from points to an axis-aligned box (min-image per axis
    when periodic)."""
    d = np.maximum(np.maximum(lo - pos, pos - hi), 0.0)
    if periodic:
        dm = np.maximum(np.maximum((lo - box) - pos, pos - (hi - box)), 0.0)
        dp = np.maximum(np.maximum((lo + box) - pos, pos - (hi + box)), 0.0)
        d = np.minimum(d, np.minimum(dm, dp))
    return np.sum(d * d, axis=1)


def hist_from_todo_sizes(todo: np.ndarray, max_iterations: int) -> np.ndarray:
    """Rounds histogram (hist[r] = particles converging in round r) of a
    todo trace; traces of disjoint target sets add as histograms."""
    hist = np.zeros(max_iterations + 2, dtype=np.int64)
    todo = np.asarray(todo, dtype=np.int64)
    nxt = np.append(todo[1:], 0)
    hist[1:len(todo) + 1] = todo - nxt
    return hist


def todo_sizes_from_hist(hist: np.ndarray) -> np.ndarray:
    """PassStats.todo_sizes from a rounds histogram (entries >= 1)."""
    last = int(np.max(np.nonzero(hist[1:-1])[0]) + 1) if hist[1:-1].any() else 0
    tail = np.cumsum(hist[::-1])[::-1]
    return tail[1:last + 1].astype(np.int64)


# ---------------------------------------------------------------------------
# per-rank compute backends
# ---------------------------------------------------------------------------
class TorchOps:
    """Record plumbing of the decomposition in plain torch ops (any device);
    the host / test backend.  ``LibCompute`` replaces every op with the
    library's kernels (csrc/sph_decomp.cu)."""

    def pack_rows(self, order, x, y, z, m, h0, gid, keys):
        import torch
        k = keys[order]
        return torch.stack([x[order].double(), y[order].double(), z[order].double(), m[order], h0[order],
                            gid[order].contiguous().view(torch.float64), (k >> 32).double(),
                            (k & 0xFFFFFFFF).double()], dim=1)

    def gather_rows(self, rows, idx):
        return rows[idx]

    def row_keys(self, rows):
        import torch
        return (rows[:, 6].to(torch.int64) << 32) | rows[:, 7].to(torch.int64)

    def level_bounds(self, keys_sorted, k, half):
        return level_bounds(keys_sorted, k, half)

    def window_bounds(self, rows, bound, k, max_abs=0.0):
        return window_bounds(rows, bound, k)

    def bbox(self, x, y, z):
        import torch
        mx = [torch.aminmax(t) for t in (x, y, z)]
        return torch.stack([v.min for v in mx] + [v.max for v in mx]).to(torch.float64)

    def ghost_mask(self, gdesc, gstart, gcount, rows, fdesc, frank, periodic, box, pair_chunk=1 << 22):
        return ghost_mask(gdesc, gstart, gcount, rows, fdesc, frank, periodic, box, pair_chunk)

    def group_boxes(self, rows, bound, starts, counts):
        import torch
        ng = starts.numel()
        gid = torch.repeat_interleave(torch.arange(ng, device=rows.device), counts)
        gidx = gid.view(-1, 1).expand(-1, 3)
        big = float(np.finfo(np.float64).max)
        pos = rows[:, :3]
        lo = torch.full((ng, 3), big, dtype=torch.float64, device=rows.device).scatter_reduce(0, gidx, pos, "amin")
        hi = torch.full((ng, 3), -big, dtype=torch.float64, device=rows.device).scatter_reduce(0, gidx, pos, "amax")
        mb = torch.zeros(ng, dtype=torch.float64, device=rows.device).scatter_reduce(0, gid, bound, "amax")
        return torch.cat([lo, hi, mb.view(-1, 1)], dim=1)


class LibCompute(TorchOps):
    """The product: libsph_b200 on this rank's GPU (device-resident arrays).
    ``decomposed_pass`` runs on the library's stream, so torch ops, NCCL and
    the library's kernels are ordered without extra synchronisation."""

    def __init__(self, device: int = 0, private_context: bool = False):
        import torch

        from . import _lib
        self.torch = torch
        self.lib = _lib
        self.L = _lib.load()
        self.device = device
        self.ctx = _lib.new_context(device) if private_context else _lib.context(device)
        self.keep_inputs = False
        self.last_inputs = None
        self.stream = torch.cuda.ExternalStream(_lib.stream_handle(self.ctx), device=f"cuda:{device}")
        self.last_stats = None

    def _ck(self, rc, what):
        if rc != self.lib.SPH_OK:
            raise RuntimeError(f"{what} failed ({rc}): {self.lib.last_error(self.ctx)}")

    @staticmethod
    def _p(t):
        import ctypes
        return ctypes.c_void_p(t.data_ptr())

    def _sync_in(self, dev):
        cur = self.torch.cuda.current_stream(dev)
        if cur.cuda_stream != self.stream.cuda_stream:
            self.stream.wait_stream(cur)
        return cur

    def _sync_out(self, cur):
        if cur.cuda_stream != self.stream.cuda_stream:
            cur.wait_stream(self.stream)

    def keys(self, x, y, z, centre, half):
        import ctypes
        torch = self.torch
        n = x.numel()
        out = torch.empty(n, dtype=torch.int64, device=x.device)
        if n == 0:
            return out
        prec = self.lib.PRECISION["f32" if x.dtype == torch.float32 else "f64"]
        c3 = (ctypes.c_double * 3)(*[float(v) for v in centre])
        cur = self._sync_in(x.device)
        self._ck(self.L.sph_morton_keys_device(self.ctx, prec, n, self._p(x), self._p(y), self._p(z), c3,
                                               float(half), self._p(out)), "sph_morton_keys_device")
        self._sync_out(cur)
        return out

    def pack_rows(self, order, x, y, z, m, h0, gid, keys):
        torch = self.torch
        n = order.numel()
        rows = torch.empty((n, 8), dtype=torch.float64, device=x.device)
        if n == 0:
            return rows
        prec = self.lib.PRECISION["f32" if x.dtype == torch.float32 else "f64"]
        cur = self._sync_in(x.device)
        self._ck(self.L.sph_decomp_pack_rows_device(self.ctx, prec, n, self._p(order), self._p(x), self._p(y),
                                                    self._p(z), self._p(m), self._p(h0), self._p(gid),
                                                    self._p(keys), self._p(rows)), "sph_decomp_pack_rows_device")
        self._sync_out(cur)
        return rows

    def gather_rows(self, rows, idx):
        torch = self.torch
        n = idx.numel()
        out = torch.empty((n, rows.shape[1]), dtype=torch.float64, device=rows.device)
        if n == 0:
            return out
        cur = self._sync_in(rows.device)
        self._ck(self.L.sph_decomp_gather_rows_device(self.ctx, n, rows.shape[1], self._p(idx), self._p(rows),
                                                      self._p(out)), "sph_decomp_gather_rows_device")
        self._sync_out(cur)
        return out

    def row_keys(self, rows):
        torch = self.torch
        n = rows.shape[0]
        out = torch.empty(n, dtype=torch.int64, device=rows.device)
        if n == 0:
            return out
        cur = self._sync_in(rows.device)
        self._ck(self.L.sph_decomp_row_keys_device(self.ctx, n, self._p(rows), self._p(out)),
                 "sph_decomp_row_keys_device")
        self._sync_out(cur)
        return out

    def level_bounds(self, keys_sorted, k, half):
        torch = self.torch
        n = keys_sorted.numel()
        out = torch.empty(n, dtype=torch.float64, device=keys_sorted.device)
        if n == 0:
            return out
        cur = self._sync_in(keys_sorted.device)
        self._ck(self.L.sph_decomp_level_bounds_device(self.ctx, n, k, self._p(keys_sorted), float(half),
                                                       self._p(out)), "sph_decomp_level_bounds_device")
        self._sync_out(cur)
        return out

    def window_bounds(self, rows, bound, k, max_abs=0.0):
        n = rows.shape[0]
        if n == 0:
            return bound
        cur = self._sync_in(rows.device)
        self._ck(self.L.sph_decomp_window_bounds_device(self.ctx, n, k, rows.shape[1], self._p(rows), float(max_abs),
                                                        self._p(bound)), "sph_decomp_window_bounds_device")
        self._sync_out(cur)
        return bound

    def bbox(self, x, y, z):
        torch = self.torch
        out = torch.empty(6, dtype=torch.float64, device=x.device)
        prec = self.lib.PRECISION["f32" if x.dtype == torch.float32 else "f64"]
        cur = self._sync_in(x.device)
        self._ck(self.L.sph_bbox_device(self.ctx, prec, x.numel(), self._p(x), self._p(y), self._p(z), self._p(out)),
                 "sph_bbox_device")
        self._sync_out(cur)
        return out

    def ghost_mask(self, gdesc, gstart, gcount, rows, fdesc, frank, periodic, box, pair_chunk=1 << 22):
        torch = self.torch
        mask = torch.zeros(rows.shape[0], dtype=torch.int32, device=rows.device)
        if gdesc.shape[0] == 0 or fdesc.shape[0] == 0:
            return mask
        fr = frank.to(torch.int32).contiguous()
        fd = fdesc.contiguous()
        gd = gdesc.contiguous()
        if self.keep_inputs:
            self.last_ghost_inputs = (gd, gstart, gcount, rows, fd, fr, periodic, box)
        cur = self._sync_in(rows.device)
        self._ck(self.L.sph_decomp_ghost_mask_device(self.ctx, gd.shape[0], self._p(gd), self._p(gstart),
                                                     self._p(gcount), rows.shape[1], self._p(rows), fd.shape[0],
                                                     self._p(fd), self._p(fr), 1 if periodic else 0, float(box),
                                                     self._p(mask)), "sph_decomp_ghost_mask_device")
        self._sync_out(cur)
        return mask

    def group_boxes(self, rows, bound, starts, counts):
        torch = self.torch
        ng = starts.numel()
        out = torch.empty((ng, 7), dtype=torch.float64, device=rows.device)
        if ng == 0:
            return out
        cur = self._sync_in(rows.device)
        self._ck(self.L.sph_decomp_group_boxes_device(self.ctx, ng, self._p(starts), self._p(counts), rows.shape[1],
                                                      self._p(rows), self._p(bound), self._p(out)),
                 "sph_decomp_group_boxes_device")
        self._sync_out(cur)
        return out

    def local_pass(self, x, y, z, m, h0_t, k, n_targets, periodic, box, max_iterations):
        from .density import _raise_for
        torch = self.torch
        n = x.numel()
        prec = "f32" if x.dtype == torch.float32 else "auto"
        h = h0_t.to(torch.float64).clone()
        rho = torch.empty(n_targets, dtype=torch.float64, device=x.device)
        flags = torch.empty(n_targets, dtype=torch.uint8, device=x.device)
        prm = self.lib.SphParams(n=n, k=k, max_iterations=max_iterations, precision=self.lib.PRECISION[prec],
                                 periodic=1 if periodic else 0, box=float(box), kernel=0, reserved=0,
                                 n_targets=0 if n_targets == n else n_targets)
        if self.keep_inputs:
            self.last_inputs = (x, y, z, m, h0_t.clone(), k, n_targets, periodic, box, max_iterations)
        st = self.lib.SphStats()
        cur = self._sync_in(x.device)
        rc = self.L.sph_density_pass_device(self.ctx, prm, self._p(x), self._p(y), self._p(z), self._p(m),
                                            self._p(h), self._p(rho), self._p(flags), st)
        self._sync_out(cur)
        _raise_for(rc, self.ctx)
        self.last_stats = st.as_dict()
        todo = np.array(self.last_stats["todo_sizes"], dtype=np.int64)
        return h, rho, todo


class NumpyCompute(TorchOps):
    """A host pass (numpy arrays in and out) behind the same interface; the
    CPU tests plug the oracle in here."""

    stream = None

    def __init__(self, local_pass):
        self.fn = local_pass

    def keys(self, x, y, z, centre, half):
        import torch
        pos = np.column_stack([x.double().cpu().numpy(), y.double().cpu().numpy(), z.double().cpu().numpy()])
        return torch.from_numpy(morton_keys(pos, centre, half).astype(np.int64)).to(x.device)

    def local_pass(self, x, y, z, m, h0_t, k, n_targets, periodic, box, max_iterations):
        import torch
        a = [t.double().cpu().numpy() for t in (x, y, z, m, h0_t)]
        h, rho, todo = self.fn(*a, k, n_targets, periodic, box, max_iterations)
        return (torch.from_numpy(np.asarray(h, np.float64)).to(x.device),
                torch.from_numpy(np.asarray(rho, np.float64)).to(x.device), np.asarray(todo, np.int64))


# ---------------------------------------------------------------------------
# the decomposition
# ---------------------------------------------------------------------------
@dataclass
class DecompResult:
    gid: object           # global ids of the owned particles (tensor, int64)
    h: object             # converged smoothing length (tensor, f64)
    rho: object           # density (tensor, f64)
    todo_hist: np.ndarray  # this rank's rounds histogram (add over ranks -> PassStats.todo_sizes)
    n_owned: int
    n_ghosts: int
    max_bound: float
    bound: object = None   # the per-owned-particle bound on h (diagnostics)


def _comm_device(dist, t):
    """gloo moves host tensors; NCCL (and in-process ranks) device tensors."""
    return "cpu" if dist.get_backend() == "gloo" else t.device


def _exchange(dist, rows, send_counts):
    """All-to-all of row blocks: rows[sum(send_counts[:q]) : ...] go to rank q."""
    import torch
    cdev = _comm_device(dist, rows)
    sc = send_counts.to(device=cdev, dtype=torch.int64)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc)
    sl, rl = torch.stack([sc, rc]).cpu().tolist()  # one host round trip
    width = rows.shape[1]
    recv = torch.empty(int(sum(rl)) * width, dtype=rows.dtype, device=cdev)
    dist.all_to_all_single(recv, rows.reshape(-1).to(cdev), output_split_sizes=[c * width for c in rl],
                           input_split_sizes=[c * width for c in sl])
    return recv.to(rows.device).reshape(-1, width)


def _all_gather_var(dist, t, world):
    """all-gather of a 2-D tensor whose row count differs per rank."""
    import torch
    cdev = _comm_device(dist, t)
    cnt = torch.tensor([t.shape[0]], dtype=torch.int64, device=cdev)
    cnts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(cnts, cnt)
    cnts = torch.cat(cnts).cpu().tolist()  # one host round trip
    mx = max(max(cnts), 1)
    pad = torch.zeros((mx, t.shape[1]), dtype=t.dtype, device=cdev)
    pad[:t.shape[0]] = t.to(cdev)
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad)
    return [o[:c].to(t.device) for o, c in zip(outs, cnts)]


def level_bounds(keys_sorted, k: int, half: float):
    """Per particle (key order) a guaranteed upper bound of its K-th neighbour
    distance among these particles: sqrt(3) x the side of the deepest key cube
    holding it together with >= K others (inf when there are <= K particles).
    torch restatement of k_level_bounds (csrc/sph_decomp.cu)."""
    import torch
    n = keys_sorted.numel()
    dev = keys_sorted.device
    w = k + 1
    if n < w:
        return torch.full((n,), float("inf"), dtype=torch.float64, device=dev)
    a = keys_sorted[: n - w + 1]
    b = keys_sorted[w - 1:]
    # deepest common level of each window of K+1 consecutive keys
    lvl = torch.zeros(n - w + 1, dtype=torch.int64, device=dev)
    for level in range(1, KEY_LEVELS + 1):
        sh = 63 - 3 * level
        lvl += ((a >> sh) == (b >> sh)).to(torch.int64)
    # a particle's level = the max over the windows containing it
    padv = torch.full((w - 1,), -1, dtype=torch.int64, device=dev)
    lv = torch.cat([padv, lvl, padv]).to(torch.float32).view(1, 1, -1)
    lvp = torch.nn.functional.max_pool1d(lv, kernel_size=w, stride=1).view(-1).to(torch.int64)
    side = (2.0 * half) * torch.pow(torch.tensor(0.5, dtype=torch.float64, device=dev), lvp.to(torch.float64))
    return side * (_SQRT3 * (1.0 + 1e-9))


def window_bounds(rows, bound, k: int, bins: int = 64):
    """min(bound, an upper bound of the K-th neighbour distance from the 2W
    key-consecutive records around p, W = 3K/2): the d2 of those records
    binned linearly over [0, bound^2] (records beyond dropped), the upper
    edge of the bin holding their K-th smallest, one bin of rounding margin --
    the algorithm of k_window_bounds (csrc/sph_decomp.cu) in fp64."""
    import torch
    n = rows.shape[0]
    if n <= k:
        return bound
    w = (3 * k + 1) // 2
    pos = rows[:, :3]
    p = torch.arange(n, device=rows.device)
    s0 = torch.clamp(torch.clamp(p - w, max=n - 1 - 2 * w), min=0)
    e0 = torch.clamp(s0 + 2 * w, max=n - 1)
    cols = []
    for j in range(2 * w + 1):
        q = s0 + j
        valid = (q <= e0) & (q != p)
        d = pos[torch.clamp(q, max=n - 1)] - pos
        d2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
        cols.append(torch.where(valid, d2, torch.full_like(d2, -1.0)))
    d2 = torch.stack(cols, dim=1)
    top = torch.clamp(bound * bound, max=3.0e38)
    ok = top > 0
    safe = torch.where(ok, top, torch.ones_like(top))
    bq = torch.clamp((d2 / safe[:, None] * float(bins)).to(torch.int64), max=bins)
    bq = torch.where(d2 >= 0, bq, torch.full_like(bq, bins))  # excluded slots and records beyond the bound
    counts = torch.zeros((n, bins + 1), dtype=torch.int64, device=rows.device)
    counts.scatter_add_(1, bq, torch.ones_like(bq))
    cum = torch.cumsum(counts[:, :bins], dim=1)
    first = torch.where(cum[:, -1] >= k, torch.argmax((cum >= k).to(torch.int64), dim=1),
                        torch.full_like(cum[:, -1], bins))
    e2 = ((first + 2).to(torch.float64) / float(bins)) * top
    cand = torch.sqrt(e2) * (1.0 + 1e-9)
    use = ok & (first < bins - 1)
    return torch.where(use, torch.minimum(bound, cand), bound)


def ghost_mask(gdesc, gstart, gcount, rows, fdesc, frank, periodic, box, pair_chunk=1 << 22):
    """Bit q of mask[i]: particle i lies within a group of rank q's margin of
    that group's box -- torch restatement of k_ghost_mask (csrc/sph_decomp.cu)."""
    import torch
    dev = rows.device
    n = rows.shape[0]
    mask = torch.zeros(n, dtype=torch.int64, device=dev)
    ng, nf = gdesc.shape[0], fdesc.shape[0]
    if ng == 0 or nf == 0:
        return mask.to(torch.int32)
    flo, fhi = fdesc[:, :3], fdesc[:, 3:6]
    fm2 = (fdesc[:, 6] * (1.0 + 1e-9)) ** 2
    mlo, mhi = gdesc[:, :3], gdesc[:, 3:6]
    opos = rows[:, :3]
    step = max(1, pair_chunk // nf)
    for g0 in range(0, ng, step):
        g1 = min(ng, g0 + step)
        d2 = _gap2(mlo[g0:g1, None, :], mhi[g0:g1, None, :], flo[None], fhi[None], periodic, box)
        gi, fi = torch.nonzero(d2 <= fm2[None], as_tuple=True)
        if gi.numel() == 0:
            continue
        gi = gi + g0
        cnt = gcount[gi]
        pidx = torch.repeat_interleave(gstart[gi], cnt)
        within = torch.arange(pidx.numel(), device=dev) - torch.repeat_interleave(torch.cumsum(cnt, 0) - cnt, cnt)
        pidx = pidx + within
        fi = torch.repeat_interleave(fi, cnt)
        p = opos[pidx]
        keep = _gap2(p, p, flo[fi], fhi[fi], periodic, box) <= fm2[fi]
        for q in torch.unique(frank[fi][keep]).tolist():  # ranks < 32: one bit each
            mask[pidx[keep & (frank[fi] == q)]] |= 1 << int(q)
    return mask.to(torch.int32)


def _gap2(alo, ahi, blo, bhi, periodic, box):
    """Squared distance between boxes [alo, ahi] and [blo, bhi] (rows
    broadcast), min-image per axis when periodic."""
    import torch
    d = torch.clamp(torch.maximum(blo - ahi, alo - bhi), min=0.0)
    if periodic:
        dm = torch.clamp(torch.maximum((blo - box) - ahi, alo - (bhi - box)), min=0.0)
        dp = torch.clamp(torch.maximum((blo + box) - ahi, alo - (bhi + box)), min=0.0)
        d = torch.minimum(d, torch.minimum(dm, dp))
    return (d * d).sum(dim=-1)


def decomposed_pass(x, y, z, mass, h0, gid, k: int, compute, *, periodic: bool = False, box: float = 0.0,
                    samples: int = 1024, max_iterations: int = 100, group_particles: int = 256,
                    pair_chunk: int = 1 << 22, comm=None) -> DecompResult:
    """Collective call: every rank passes its local particles (any split) as
    1-D tensors on its compute device (positions f32 or f64, mass/h0 f64,
    gid int64).  Returns the owned particles' global ids, h and rho.
    ``comm`` defaults to torch.distributed (``ThreadComm``: in-process ranks)."""
    import contextlib

    import torch
    if comm is None:
        import torch.distributed as comm
    stream = getattr(compute, "stream", None)
    ctxm = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    caller = torch.cuda.current_stream(x.device) if stream is not None else None
    if caller is not None and caller.cuda_stream != stream.cuda_stream:
        # the inputs may still be in flight on the caller's stream (e.g. a
        # non_blocking host copy): the library's stream waits for them, and
        # their memory is not reused before the library's stream is done
        stream.wait_stream(caller)
        for t in (x, y, z, mass, h0, gid):
            if t.is_cuda:
                t.record_stream(stream)
    with ctxm:
        res = _decomposed(x, y, z, mass, h0, gid, k, compute, periodic, box, samples, max_iterations,
                          group_particles, pair_chunk, comm)
    if caller is not None and caller.cuda_stream != stream.cuda_stream:
        # the results were produced on the library's stream: order the caller's
        # stream after it, and keep their memory from being reused too early
        caller.wait_stream(stream)
        for t in (res.gid, res.h, res.rho, res.bound):
            if t is not None and t.is_cuda:
                t.record_stream(caller)
    return res


class ThreadComm:
    """The collectives of ``decomposed_pass`` between ranks that are threads
    of one process (one shared ``ThreadWorld``): checks the decomposition at
    world sizes beyond the GPUs at hand.  Host-side barriers only; no kernel
    waits on another rank."""

    def __init__(self, world_state, rank: int):
        import torch.distributed as tdist
        self.W = world_state
        self.rank = rank
        self.ReduceOp = tdist.ReduceOp

    def get_rank(self):
        return self.rank

    def get_world_size(self):
        return self.W.world

    def get_backend(self):
        return "thread"

    def _swap(self, obj):
        import torch
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()
        self.W.slots[self.rank] = obj
        self.W.barrier.wait()
        vals = list(self.W.slots)
        self.W.barrier.wait()
        return vals

    def all_reduce(self, t, op=None):
        import torch
        vals = self._swap(t.clone())
        st = torch.stack([v.to(t.device) for v in vals])
        if op is None or op == self.ReduceOp.SUM:
            r = st.sum(0)
        elif op == self.ReduceOp.MAX:
            r = st.max(0).values
        else:
            r = st.min(0).values
        t.copy_(r)

    def all_gather(self, outs, t):
        vals = self._swap(t.clone())
        for o, v in zip(outs, vals):
            o.copy_(v.to(o.device))

    def all_to_all_single(self, out, inp, output_split_sizes=None, input_split_sizes=None):
        import torch
        w = self.W.world
        if input_split_sizes is None:
            input_split_sizes = [inp.numel() // w] * w
        chunks = [c.clone() for c in torch.split(inp, input_split_sizes)]
        vals = self._swap(chunks)
        got = [vals[q][self.rank].to(out.device) for q in range(w)]
        out.copy_(torch.cat(got) if got else out)


class ThreadWorld:
    def __init__(self, world: int):
        import threading
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


def _decomposed(x, y, z, mass, h0, gid, k, compute, periodic, box, samples, max_iterations, group_particles,
                pair_chunk, dist):
    import os
    import time

    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = x.device
    pdt = x.dtype
    f64 = torch.float64
    n_local = x.numel()
    cdev = _comm_device(dist, x)
    _tm = [] if os.environ.get("SPH_DECOMP_TIMING") else None

    def mark(name):
        if _tm is not None:
            if dev.type == "cuda":
                torch.cuda.synchronize(dev)
            _tm.append((name, time.perf_counter()))
    mark("start")

    # 1. common root cube; global particle count
    big = float(np.finfo(np.float64).max)
    if n_local:
        bb = compute.bbox(x, y, z)
        lo, hi = bb[:3], bb[3:]
    else:
        lo = torch.full((3,), big, dtype=f64, device=dev)
        hi = torch.full((3,), -big, dtype=f64, device=dev)
    mm = torch.cat([-lo, hi]).to(cdev)
    dist.all_reduce(mm, op=dist.ReduceOp.MAX)
    mm = mm.cpu().numpy()  # one host round trip (the particle count travels with the key samples)
    centre, half = root_cube(-mm[:3], mm[3:6])
    mark("bbox")

    # 2. keys, splitters, key-sorted records, redistribution
    keys = compute.keys(x, y, z, centre, half)
    sk, order = torch.sort(keys)
    if n_local:
        idx = torch.linspace(0, n_local - 1, samples, device=dev).round().to(torch.int64)
        mine = sk[idx]
    else:
        mine = torch.full((samples,), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)
    mine = torch.cat([mine, torch.full((1,), n_local, dtype=torch.int64, device=dev)])
    gathered = [torch.empty(samples + 1, dtype=torch.int64, device=cdev) for _ in range(world)]
    dist.all_gather(gathered, mine.to(cdev))
    gk = torch.stack(gathered)
    n_total_d = gk[:, samples].sum()
    # count-weighted splitters: each of rank q's samples stands for n_q /
    # samples particles, so uneven (or empty) ranks do not bias the cuts
    sk_all, so = torch.sort(gk[:, :samples].reshape(-1))
    wts = (gk[:, samples].to(f64) / samples).view(-1, 1).expand(-1, samples).reshape(-1)[so]
    cum = torch.cumsum(wts, 0)
    goal = torch.arange(1, world, device=cum.device, dtype=f64) * (n_total_d.to(f64) / world)
    pick = torch.clamp(torch.searchsorted(cum, goal), max=max(sk_all.numel() - 1, 0))
    splitters = sk_all[pick].to(dev)
    cuts = torch.searchsorted(sk, splitters)  # rank q owns keys in [splitter[q-1], splitter[q])
    edges = torch.cat([torch.zeros(1, dtype=torch.int64, device=dev), cuts,
                       torch.full((1,), n_local, dtype=torch.int64, device=dev)])
    rows = compute.pack_rows(order, x, y, z, mass.to(f64), h0.to(f64), gid.to(torch.int64), keys)
    n_total = int(n_total_d)
    mark("keys+pack")
    recv = _exchange(dist, rows, edges[1:] - edges[:-1])
    mark("redistribute")
    okeys, o2 = torch.sort(compute.row_keys(recv), stable=True)
    owned = compute.gather_rows(recv, o2)

    n_own = owned.shape[0]
    mark("sort owned")

    # 3. bounds, 4. descriptors (groups of a coarse key prefix)
    max_abs = float(np.max(np.abs(centre)) + half)
    bound = compute.window_bounds(owned, compute.level_bounds(okeys, k, half), k, max_abs)
    gl = int(min(KEY_LEVELS, max(1, round(math.log(max(n_total / group_particles, 1.0), 8)))))
    if n_own:
        # a descriptor = <= group_particles consecutive records of one key cube
        pref = okeys >> (63 - 3 * gl)
        newg = torch.ones(n_own, dtype=torch.bool, device=dev)
        newg[1:] = pref[1:] != pref[:-1]
        newg[::group_particles] = True  # and at most group_particles records each
        gstart = torch.nonzero(newg).view(-1)
        gcnt = torch.diff(torch.cat([gstart, torch.full((1,), n_own, dtype=torch.int64, device=dev)]))
        desc = compute.group_boxes(owned, bound, gstart, gcnt)
    else:
        desc = torch.zeros((0, 7), dtype=f64, device=dev)
        gcnt = torch.zeros(0, dtype=torch.int64, device=dev)
        gstart = gcnt
    descs = _all_gather_var(dist, desc, world)
    mark("bounds+descriptors")

    # 5. ghosts: my particles within a peer group's bound of that group's box
    if world > 32:
        raise ValueError("the ghost masks hold up to 32 ranks")
    fr = [d for q, d in enumerate(descs) if q != rank]
    if fr and n_own:
        fdesc = torch.cat(fr)
        frank = torch.cat([torch.full((d.shape[0],), q, dtype=torch.int32, device=dev)
                           for q, d in enumerate(descs) if q != rank])
        mask = compute.ghost_mask(desc, gstart, gcnt, owned, fdesc, frank, periodic, box)
        # (rank, particle) pairs grouped by rank: one nonzero over the rank bits
        bits = (mask.view(1, -1) >> torch.arange(world, device=dev, dtype=mask.dtype).view(-1, 1)) & 1
        nz = torch.nonzero(bits)
        gp = nz[:, 1]
        gcounts = torch.bincount(nz[:, 0], minlength=world)
    else:
        gp = torch.zeros(0, dtype=torch.int64, device=dev)
        gcounts = torch.zeros(world, dtype=torch.int64, device=dev)
    mark("ghost select")
    ghosts = _exchange(dist, compute.gather_rows(owned, gp), gcounts)
    mark("ghost exchange")

    # 6. final pass: owned targets first, then ghosts
    allp = torch.cat([owned, ghosts]) if ghosts.shape[0] else owned
    if n_own:
        ax, ay, az = (allp[:, i].to(pdt).contiguous() for i in range(3))
        h, rho, todo = compute.local_pass(ax, ay, az, allp[:, 3].contiguous(), owned[:, 4].contiguous(), k,
                                          n_own, periodic, box, max_iterations)
    else:
        h = rho = torch.zeros(0, dtype=f64, device=dev)
        todo = np.zeros(0, dtype=np.int64)
    mark("final pass")
    if _tm is not None and rank == 0:
        print("[decomp] " + " ".join(f"{_tm[i][0]} {1e3 * (_tm[i][1] - _tm[i - 1][1]):.2f}"
                                     for i in range(1, len(_tm))), flush=True)
    hist = hist_from_todo_sizes(np.asarray(todo, dtype=np.int64), max_iterations)
    mb = float(bound.max().item()) if n_own else 0.0
    # the global id rides in column 5 as its int64 bit pattern (exact for any id)
    return DecompResult(gid=owned[:, 5].contiguous().view(torch.int64), h=h, rho=rho, todo_hist=hist, n_owned=n_own,
                        n_ghosts=int(ghosts.shape[0]), max_bound=mb, bound=bound)


# ---------------------------------------------------------------------------
# numpy front end (host arrays in and out)
# ---------------------------------------------------------------------------
@dataclass
class DistResult:
    gid: np.ndarray
    h: np.ndarray
    rho: np.ndarray
    todo_hist: np.ndarray
    n_ghosts: int
    margin: float


def density_pass_distributed(x, y, z, mass, h0, gid, k: int, local_pass, *, periodic: bool = False,
                             box: float = 0.0, samples: int = 1024, device="cpu",
                             max_iterations: int = 100) -> DistResult:
    """``decomposed_pass`` on host arrays.  ``local_pass`` is either a host
    function ``(x, y, z, mass, h0_targets, k, n_targets, periodic, box,
    max_iterations) -> (h, rho, todo_sizes)`` (numpy) or a compute backend
    (``LibCompute``)."""
    import torch
    compute = local_pass if hasattr(local_pass, "local_pass") else NumpyCompute(local_pass)
    if isinstance(compute, LibCompute):
        device = f"cuda:{compute.device}"
    xa = np.asarray(x)
    pdt = torch.float32 if xa.dtype == np.float32 else torch.float64

    def t(a, dt):
        return torch.as_tensor(np.ascontiguousarray(a)).to(device=device, dtype=dt)

    r = decomposed_pass(t(x, pdt), t(y, pdt), t(z, pdt), t(mass, torch.float64), t(h0, torch.float64),
                        t(gid, torch.int64), k, compute, periodic=periodic, box=box, samples=samples,
                        max_iterations=max_iterations)
    return DistResult(gid=r.gid.cpu().numpy(), h=r.h.cpu().numpy(), rho=r.rho.cpu().numpy(),
                      todo_hist=r.todo_hist, n_ghosts=r.n_ghosts, margin=r.max_bound)


def gpu_local_pass(device: int = 0):
    """The product per-rank compute: libsph_b200 on this rank's GPU."""
    return LibCompute(device)
