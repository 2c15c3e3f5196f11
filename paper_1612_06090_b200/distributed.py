"""Domain-decomposed density pass over P ranks (one process per GPU).

The reference runs on one shared-memory node (threads, scheduler.py of the
reference); it has no distributed mode.  Here each rank owns a contiguous
range of the same 63-bit x-major Morton keys the ordering uses (the key of a
particle is the reference octree path, octree.py:93-104), so a rank's
particles form a compact piece of space.  The exchange steps:

  1. bbox all-reduce (MIN / MAX) -> the common root cube (octree.py:324-328)
  2. key splitters from an all-gather of evenly spaced key samples
     (count-balanced), then an all-to-all that moves every particle record
     (x, y, z, m, h0, global id) to its owner
  3. a local pass over owned particles only gives h_local >= h (a K-th
     neighbour among a subset is never nearer): per rank, the ghost margin
     m_r = max h_local is a guaranteed cover.  Ghosts = every particle
     within m_r of rank r's box (min-image distance when periodic), sent
     with a second all-to-all
  4. the final pass over owned + ghosts with the owned particles as targets
     (sph_params.n_targets) is exact: each target sees every particle within
     its true h, so h is bit-identical to the single-GPU result and the todo
     trace (a function of h0 and d2_K) is too.

Collectives go through torch.distributed: NCCL (device tensors over
NVLink/NVSwitch) on GPUs, gloo on CPU (tests).  ``local_pass`` is the
per-rank compute; ``gpu_local_pass`` is the product one, the tests pass the
CPU oracle instead to check the decomposition logic without GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KEY_LEVELS = 21


def root_cube(lo: np.ndarray, hi: np.ndarray):
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
        # distance to the box images shifted by +-box along each axis
        dm = np.maximum(np.maximum((lo - box) - pos, pos - (hi - box)), 0.0)
        dp = np.maximum(np.maximum((lo + box) - pos, pos - (hi + box)), 0.0)
        d = np.minimum(d, np.minimum(dm, dp))
    return np.sum(d * d, axis=1)


@dataclass
class DistResult:
    gid: np.ndarray       # global ids of the particles this rank owns
    h: np.ndarray         # converged smoothing length
    rho: np.ndarray       # density
    todo_hist: np.ndarray  # reference rounds histogram contribution (PassStats.todo_sizes by sum)
    n_ghosts: int
    margin: float


def _torch():
    import torch
    import torch.distributed as dist
    return torch, dist


def _all_to_all_rows(rows: np.ndarray, dest: np.ndarray, world: int, device) -> np.ndarray:
    """Send row i to rank dest[i]; returns the rows received (float64)."""
    torch, dist = _torch()
    order = np.argsort(dest, kind="stable")
    rows = np.ascontiguousarray(rows[order])
    send_counts = np.bincount(dest, minlength=world).astype(np.int64)
    sc = torch.from_numpy(send_counts).to(device)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc)
    recv_counts = rc.cpu().numpy()
    width = rows.shape[1] if rows.ndim == 2 else 1
    send = torch.from_numpy(rows.reshape(-1)).to(device)
    recv = torch.empty(int(recv_counts.sum()) * width, dtype=torch.float64, device=device)
    dist.all_to_all_single(recv, send, output_split_sizes=(recv_counts * width).tolist(),
                           input_split_sizes=(send_counts * width).tolist())
    return recv.cpu().numpy().reshape(-1, width)


def density_pass_distributed(x, y, z, mass, h0, gid, k: int, local_pass, *, periodic: bool = False,
                             box: float = 0.0, samples: int = 1024, device="cpu",
                             max_iterations: int = 100) -> DistResult:
    """Collective call: every rank passes its local particles (any split).

    ``local_pass(x, y, z, mass, h0_targets, k, n_targets, periodic, box,
    max_iterations) -> (h, rho, todo_sizes)`` computes the targets
    [0, n_targets) of the arrays it is given (the rest are ghosts);
    ``todo_sizes`` is the reference todo trace over those targets.
    """
    torch, dist = _torch()
    rank, world = dist.get_rank(), dist.get_world_size()
    pos = np.column_stack([np.asarray(x, np.float64), np.asarray(y, np.float64), np.asarray(z, np.float64)])
    n_local = pos.shape[0]

    # 1. common root cube
    big = np.finfo(np.float64).max
    lo = torch.tensor(pos.min(axis=0) if n_local else np.full(3, big), dtype=torch.float64, device=device)
    hi = torch.tensor(pos.max(axis=0) if n_local else np.full(3, -big), dtype=torch.float64, device=device)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX)
    centre, half = root_cube(lo.cpu().numpy(), hi.cpu().numpy())

    # 2. key-range ownership from sampled splitters
    keys = morton_keys(pos, centre, half)
    sk = np.sort(keys)
    if n_local:
        idx = np.linspace(0, n_local - 1, samples).astype(np.int64)
        mine = sk[idx].astype(np.int64)  # keys < 2^63: exact in int64
    else:
        mine = np.full(samples, np.iinfo(np.int64).max, dtype=np.int64)
    t = torch.from_numpy(mine).to(device)
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    allk = np.sort(np.concatenate([g.cpu().numpy() for g in gathered]))
    splitters = allk[(np.arange(1, world) * allk.size) // world].astype(np.uint64)
    dest = np.searchsorted(splitters, keys, side="right").astype(np.int64)
    rows = np.column_stack([pos, np.asarray(mass, np.float64), np.asarray(h0, np.float64),
                            np.asarray(gid, np.float64)])
    owned = _all_to_all_rows(rows, dest, world, device)
    owned = owned[np.argsort(owned[:, 5], kind="stable")]  # deterministic order: by global id
    n_own = owned.shape[0]

    # 3. local pass on owned particles only -> guaranteed ghost margin
    if n_own > k:
        h_loc, _, _ = local_pass(owned[:, 0], owned[:, 1], owned[:, 2], owned[:, 3], owned[:, 4], k, n_own,
                                 periodic, box, max_iterations)
        margin = float(np.max(h_loc)) if n_own else 0.0
    else:
        margin = np.inf
    if not np.isfinite(margin):
        margin = float(box) if periodic else 2.0 * half * np.sqrt(3.0) + 1.0
    olo = owned[:, :3].min(axis=0) if n_own else np.full(3, big)
    ohi = owned[:, :3].max(axis=0) if n_own else np.full(3, -big)
    info = torch.tensor(np.concatenate([olo, ohi, [margin]]), dtype=torch.float64, device=device)
    infos = [torch.empty_like(info) for _ in range(world)]
    dist.all_gather(infos, info)
    infos = [i.cpu().numpy() for i in infos]

    # ghosts: my owned particles within each peer's margin of the peer's box
    send_rows, send_dest = [], []
    for q in range(world):
        if q == rank or n_own == 0:
            continue
        qlo, qhi, qm = infos[q][:3], infos[q][3:6], infos[q][6]
        if not np.all(qlo <= qhi):
            continue
        sel = box_distance2(owned[:, :3], qlo, qhi, periodic, box) <= qm * qm * (1.0 + 1e-12)
        if sel.any():
            send_rows.append(owned[sel])
            send_dest.append(np.full(int(sel.sum()), q, dtype=np.int64))
    rows_g = np.concatenate(send_rows) if send_rows else np.zeros((0, 6))
    dest_g = np.concatenate(send_dest) if send_dest else np.zeros(0, dtype=np.int64)
    ghosts = _all_to_all_rows(rows_g, dest_g, world, device)

    # 4. final pass: owned targets + ghosts
    allp = np.concatenate([owned, ghosts]) if ghosts.size else owned
    if n_own:
        h, rho, todo = local_pass(allp[:, 0], allp[:, 1], allp[:, 2], allp[:, 3], owned[:, 4], k, n_own,
                                  periodic, box, max_iterations)
    else:
        h = rho = np.zeros(0)
        todo = np.zeros(0, dtype=np.int64)
    hist = hist_from_todo_sizes(np.asarray(todo, dtype=np.int64), max_iterations)
    return DistResult(gid=owned[:, 5].astype(np.int64), h=np.asarray(h), rho=np.asarray(rho), todo_hist=hist,
                      n_ghosts=int(ghosts.shape[0]), margin=margin)


def hist_from_todo_sizes(todo: np.ndarray, max_iterations: int) -> np.ndarray:
    """Rounds histogram (hist[r] = particles converging in round r) of a
    todo trace; traces of disjoint target sets add as histograms."""
    hist = np.zeros(max_iterations + 2, dtype=np.int64)
    nxt = np.append(todo[1:], 0)
    hist[1:len(todo) + 1] = todo - nxt
    return hist


def todo_sizes_from_hist(hist: np.ndarray) -> np.ndarray:
    """PassStats.todo_sizes from a rounds histogram (entries >= 1)."""
    last = int(np.max(np.nonzero(hist[1:-1])[0]) + 1) if hist[1:-1].any() else 0
    tail = np.cumsum(hist[::-1])[::-1]
    return tail[1:last + 1].astype(np.int64)


def gpu_local_pass(device: int = 0):
    """The product per-rank compute: libsph_b200 on this rank's GPU."""
    from .density import density_pass_soa

    def run(x, y, z, m, h0_t, k, n_targets, periodic, box, max_iterations):
        h, rho, _, st = density_pass_soa(x, y, z, m, h0_t, k, max_iterations, precision="auto",
                                         periodic=periodic, box=box, device=device, n_targets=n_targets)
        return h, rho, st.todo_sizes

    return run
