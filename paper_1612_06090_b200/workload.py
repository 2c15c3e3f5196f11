"""Seeded synthetic particle sets for the BASELINE configurations.

* ``uniform_box`` regenerates the reference's UniformBox stream bit-exactly
  (splitmix64, workload.py:42-84 of the reference): draw t (0-based, three
  per particle, x-y-z order) is ``mix(seed + (t+1)*GAMMA) >> 11`` scaled by
  2^-53 and by the box side.  The sequential stream is a pure function of
  the counter, so it vectorises.
* ``config_device`` generates configs 2-5 on the GPU (C ABI
  ``sph_nfw_positions_device``; the bench and the full-size tests use it):
  the host draws only the halo table (``halo_table``: the same rules as
  below), every per-particle draw is the splitmix64 counter stream (draw
  8i + j of particle i), so 134M particles take milliseconds.
  ``nfw_host_restatement`` is its numpy restatement (test infrastructure).
* ``nfw_halos`` is the host clustered generator (small CPU tests), which
  the reference does not have.  Rules chosen and recorded here:
  halo particle counts are drawn from dN/dM ~ M^-1.9 on [100, 50000] and
  rescaled (largest remainder) to sum to round(f_halo * N); r_vir from an
  overdensity of 200 times the mean particle density (so it scales with the
  halo's particle count); radii by inverting the NFW enclosed mass
  m(x) = ln(1+x) - x/(1+x) up to x = c; isotropic directions; periodic wrap
  into [0, L); positions rounded to fp32 when ``fp32`` is set.  Velocities
  are generated (sigma ~ M^(1/3)) but never read by the density pass.
"""

from __future__ import annotations

import math

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)
_TO_UNIT = 2.0 ** -53


def _splitmix_values(seed: int, start: int, count: int) -> np.ndarray:
    t = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + t * _GAMMA
        z = (s ^ (s >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, count: int, start: int = 0) -> np.ndarray:
    """The reference's splitmix64 uniform doubles in [0, 1)."""
    return (_splitmix_values(seed, start, count) >> np.uint64(11)).astype(np.float64) * _TO_UNIT


def uniform_box(n: int, seed: int, box: float = 1.0) -> np.ndarray:
    """(n, 3) positions identical to the reference generate(UNIFORM_BOX)."""
    u = uniform01(seed, 3 * n).reshape(n, 3)
    v = u * box
    over = v >= box
    if over.any():
        v[over] = np.nextafter(box, 0.0)
    return v


def uniform_box_device(n: int, seed: int, box: float = 1.0, device: int = 0):
    """``uniform_box`` generated on the GPU (C ABI ``sph_uniform_box_device``):
    three fp64 torch tensors (x, y, z) on ``cuda:device``, bit-exact with
    ``uniform_box`` (the on-device input path)."""
    import ctypes

    import torch

    from . import _lib

    L = _lib.load()
    ctx = _lib.context(device)
    out = [torch.empty(n, dtype=torch.float64, device=f"cuda:{device}") for _ in range(3)]
    rc = L.sph_uniform_box_device(ctx, n, ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), float(box),
                                  *[ctypes.c_void_p(t.data_ptr()) for t in out])
    if rc != _lib.SPH_OK:
        raise RuntimeError(f"sph_uniform_box_device failed ({rc}): {_lib.last_error(ctx)}")
    torch.cuda.ExternalStream(_lib.stream_handle(ctx), device=f"cuda:{device}").synchronize()
    return tuple(out)


def nfw_enclosed(x):
    return np.log1p(x) - x / (1.0 + x)


def _nfw_radii(rng, count: int, c: float, r_vir: float, x_max: float) -> np.ndarray:
    """Inverse-CDF sampling of the NFW profile truncated at x_max = r/r_s."""
    u = rng.random(count) * nfw_enclosed(x_max)
    lo = np.zeros(count)
    hi = np.full(count, x_max)
    for _ in range(60):  # bisection; m(x) is monotone
        mid = 0.5 * (lo + hi)
        below = nfw_enclosed(mid) < u
        lo = np.where(below, mid, lo)
        hi = np.where(below, hi, mid)
    return 0.5 * (lo + hi) * (r_vir / c)


def _directions(rng, count: int) -> np.ndarray:
    v = rng.normal(size=(count, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v


def _largest_remainder(weights: np.ndarray, total: int) -> np.ndarray:
    raw = weights / weights.sum() * total
    base = np.floor(raw).astype(np.int64)
    rem = total - int(base.sum())
    if rem > 0:
        order = np.argsort(-(raw - base), kind="stable")
        base[order[:rem]] += 1
    return base


def nfw_halos(n: int, box: float, n_halos: int, seed: int, concentration: float = 10.0,
              halo_fraction: float = 0.8, m_min: float = 100.0, m_max: float = 50000.0,
              slope: float = -1.9, fp32: bool = True, truncate: float = 1.0):
    """Clustered set: ``halo_fraction`` of N in NFW halos, rest uniform.

    Returns (pos (n,3) float64, vel (n,3) float32, halo_counts).
    """
    rng = np.random.default_rng(seed)
    n_halo_total = int(round(halo_fraction * n))
    # dN/dM ~ M^slope on [m_min, m_max]: inverse CDF of a power law
    a = slope + 1.0
    u = rng.random(n_halos)
    masses = (m_min ** a + u * (m_max ** a - m_min ** a)) ** (1.0 / a)
    counts = _largest_remainder(masses, n_halo_total) if n_halos else np.zeros(0, np.int64)
    mean_density = n / box ** 3
    centres = rng.random((n_halos, 3)) * box
    pos = np.empty((n, 3))
    vel = np.empty((n, 3), dtype=np.float32)
    off = 0
    for hcount, c0 in zip(counts, centres):
        if hcount == 0:
            continue
        r_vir = (3.0 * hcount / (4.0 * math.pi * 200.0 * mean_density)) ** (1.0 / 3.0)
        r = _nfw_radii(rng, int(hcount), concentration, r_vir, concentration * truncate)
        pos[off:off + hcount] = c0 + r[:, None] * _directions(rng, int(hcount))
        sigma = float(hcount) ** (1.0 / 3.0) * 0.1
        vel[off:off + hcount] = rng.normal(0.0, sigma, (hcount, 3))
        off += int(hcount)
    rest = n - off
    pos[off:] = rng.random((rest, 3)) * box
    vel[off:] = rng.normal(0.0, 1.0, (rest, 3))
    pos = np.mod(pos, box)
    if fp32:
        pos = pos.astype(np.float32).astype(np.float64)
        # fp32 rounding can land exactly on the box side
        pos[pos >= box] = np.float64(np.nextafter(np.float32(box), np.float32(0.0)))
    return pos, vel, counts


def single_halo(n: int, box: float, seed: int, concentration: float = 20.0, r_vir: float = 1.0,
                truncate: float = 2.0, background_fraction: float = 0.05, fp32: bool = True):
    """BASELINE config 5: one NFW halo at the box centre plus a background."""
    rng = np.random.default_rng(seed)
    n_bg = int(round(background_fraction * n))
    n_h = n - n_bg
    r = _nfw_radii(rng, n_h, concentration, r_vir, concentration * truncate)
    pos = np.empty((n, 3))
    pos[:n_h] = 0.5 * box + r[:, None] * _directions(rng, n_h)
    pos[n_h:] = rng.random((n_bg, 3)) * box
    pos = np.mod(pos, box)
    if fp32:
        pos = pos.astype(np.float32).astype(np.float64)
        pos[pos >= box] = np.float64(np.nextafter(np.float32(box), np.float32(0.0)))
    vel = rng.normal(0.0, 1.0, (n, 3)).astype(np.float32)
    return pos, vel


def config(number: int, seed: int | None = None):
    """Inputs of BASELINE.json config ``number`` (1-5) as a dict."""
    seed = number if seed is None else seed
    if number == 1:
        n = 32768
        pos = uniform_box(n, seed, 1.0)
        vel = np.random.default_rng(seed).normal(0.0, 1.0, (n, 3)).astype(np.float32)
        return dict(pos=pos, vel=vel, mass=np.full(n, 1.0 / n), h0=np.full(n, 2.0 * n ** (-1.0 / 3.0)),
                    k=64, box=1.0, periodic=True, fp32=False, name="C1 uniform 32768 fp64")
    if number in (2, 3, 4):
        n, box, halos = {2: (1 << 20, 100.0, 200), 3: (1 << 24, 100.0 * 16 ** (1.0 / 3.0), 20000),
                         4: (1 << 27, 400.0, 150000)}[number]
        pos, vel, _ = nfw_halos(n, box, halos, seed)
        h0 = _initial_h(box, n, 64)
        return dict(pos=pos, vel=vel, mass=np.full(n, 1.0 / n), h0=np.full(n, h0), k=64, box=box,
                    periodic=True, fp32=True, name=f"C{number} NFW {n} fp32")
    if number == 5:
        n, box = 1 << 23, 4.0
        pos, vel = single_halo(n, box, seed)
        h0 = _initial_h(box, n, 128)
        return dict(pos=pos, vel=vel, mass=np.full(n, 1.0 / n), h0=np.full(n, h0), k=128, box=box,
                    periodic=True, fp32=True, name="C5 single NFW halo 8388608 fp32")
    if number == 6:  # diagnostic (not a BASELINE config): C2's size and box, uniform
        n, box = 1 << 20, 100.0
        pos = (np.random.default_rng(seed).random((n, 3)) * box).astype(np.float32).astype(np.float64)
        pos[pos >= box] = np.float64(np.nextafter(np.float32(box), np.float32(0.0)))
        return dict(pos=pos, vel=np.zeros((n, 3), np.float32), mass=np.full(n, 1.0 / n),
                    h0=np.full(n, _initial_h(box, n, 64)), k=64, box=box, periodic=True, fp32=True,
                    name="uniform 1048576 fp32 (diagnostic)")
    raise ValueError(f"unknown config {number}")


# ---------------------------------------------------------------------------
# on-device clustered generator (C ABI sph_nfw_positions_device)
# ---------------------------------------------------------------------------
def halo_table(n: int, box: float, n_halos: int, seed: int, halo_fraction: float = 0.8,
               m_min: float = 100.0, m_max: float = 50000.0, slope: float = -1.9):
    """Halo counts, centres, r_vir and velocity sigma of ``nfw_halos`` (the
    same host rules: power-law masses rescaled by largest remainder, r_vir
    at 200x the mean density); the per-particle draws are the device's.
    Returns (start int64[n_halos + 1], halo float64[n_halos, 5])."""
    rng = np.random.default_rng(seed)
    n_halo_total = int(round(halo_fraction * n))
    a = slope + 1.0
    u = rng.random(n_halos)
    masses = (m_min ** a + u * (m_max ** a - m_min ** a)) ** (1.0 / a)
    counts = _largest_remainder(masses, n_halo_total) if n_halos else np.zeros(0, np.int64)
    centres = rng.random((n_halos, 3)) * box
    mean_density = n / box ** 3
    r_vir = (3.0 * counts / (4.0 * math.pi * 200.0 * mean_density)) ** (1.0 / 3.0)
    sigma = counts.astype(np.float64) ** (1.0 / 3.0) * 0.1
    start = np.zeros(n_halos + 1, dtype=np.int64)
    np.cumsum(counts, out=start[1:])
    halo = np.ascontiguousarray(np.column_stack([centres, r_vir, sigma]), dtype=np.float64)
    return start, halo


def nfw_device(n: int, box: float, start, halo, seed: int, concentration: float = 10.0, x_max: float | None = None,
               device: int = 0, velocities: bool = False):
    """Positions (three fp32 cuda tensors, and optionally (n, 3) fp32
    velocities) of the clustered set generated on the GPU."""
    import ctypes

    import torch

    from . import _lib

    L = _lib.load()
    ctx = _lib.context(device)
    dev = f"cuda:{device}"
    d_start = torch.from_numpy(np.ascontiguousarray(start, dtype=np.int64)).to(dev)
    d_halo = torch.from_numpy(np.ascontiguousarray(halo, dtype=np.float64).reshape(-1)).to(dev)
    torch.cuda.synchronize(device)
    out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3)]
    vel = torch.empty((n, 3), dtype=torch.float32, device=dev) if velocities else None
    n_halos = len(start) - 1
    rc = L.sph_nfw_positions_device(ctx, n, n_halos, ctypes.c_void_p(d_start.data_ptr()),
                                    ctypes.c_void_p(d_halo.data_ptr() if n_halos else 0), float(concentration),
                                    float(concentration if x_max is None else x_max),
                                    ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), float(box),
                                    *[ctypes.c_void_p(t.data_ptr()) for t in out],
                                    ctypes.c_void_p(vel.data_ptr() if vel is not None else 0))
    if rc != _lib.SPH_OK:
        raise RuntimeError(f"sph_nfw_positions_device failed ({rc}): {_lib.last_error(ctx)}")
    torch.cuda.ExternalStream(_lib.stream_handle(ctx), device=dev).synchronize()
    return (tuple(out), vel) if velocities else tuple(out)


def nfw_host_restatement(n: int, box: float, start, halo, seed: int, concentration: float = 10.0,
                         x_max: float | None = None) -> np.ndarray:
    """numpy restatement of the device generator (same counters and formulas;
    libm may differ from the device's in the last bits of log1p / sincos, so
    a few fp32 positions can differ by an ulp).  Test infrastructure."""
    x_max = concentration if x_max is None else x_max
    i = np.arange(n, dtype=np.uint64)

    def u(j):
        t = i * np.uint64(8) + np.uint64(j + 1)
        with np.errstate(over="ignore"):
            s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + t * _GAMMA
            z = (s ^ (s >> np.uint64(30))) * _MIX1
            z = (z ^ (z >> np.uint64(27))) * _MIX2
            z = z ^ (z >> np.uint64(31))
        return (z >> np.uint64(11)).astype(np.float64) * _TO_UNIT

    start = np.asarray(start, dtype=np.int64)
    halo = np.asarray(halo, dtype=np.float64).reshape(-1, 5)
    nh = int(start[-1])
    pos = np.empty((n, 3))
    if nh:
        hid = np.searchsorted(start, np.arange(nh), side="right") - 1
        hp = halo[hid]
        um = u(0)[:nh] * nfw_enclosed(x_max)
        a = np.zeros(nh)
        b = np.full(nh, x_max)
        for _ in range(60):
            mid = 0.5 * (a + b)
            below = nfw_enclosed(mid) < um
            a = np.where(below, mid, a)
            b = np.where(below, b, mid)
        r = 0.5 * (a + b) * (hp[:, 3] / concentration)
        mu = 2.0 * u(1)[:nh] - 1.0
        phi = 6.283185307179586 * u(2)[:nh]
        s = np.sqrt(np.maximum(0.0, 1.0 - mu * mu))
        pos[:nh, 0] = hp[:, 0] + r * (s * np.cos(phi))
        pos[:nh, 1] = hp[:, 1] + r * (s * np.sin(phi))
        pos[:nh, 2] = hp[:, 2] + r * mu
    for ax in range(3):
        pos[nh:, ax] = u(ax)[nh:] * box
    pos = np.mod(pos, box).astype(np.float32)
    top = np.nextafter(np.float32(box), np.float32(0.0))
    pos[pos.astype(np.float64) >= box] = top
    return pos


def _config_table(number: int, n_ranks: int = 1):
    """(n, box, n_halos, K, concentration, x_max, halo fraction) of config 2-5."""
    g = n_ranks ** (1.0 / 3.0)
    if number in (2, 3, 4):
        n, box, halos = {2: (1 << 20, 100.0, 200), 3: (1 << 24, 100.0 * 16 ** (1.0 / 3.0), 20000),
                         4: (1 << 27, 400.0, 150000)}[number]
        return n * n_ranks, box * g, halos * n_ranks, 64, 10.0, 10.0
    if number == 5:
        return (1 << 23) * n_ranks, 4.0 * g, 1, 128, 20.0, 40.0
    raise ValueError(f"config {number} is not a clustered config")


def config_device(number: int, seed: int | None = None, device: int = 0, n_ranks: int = 1,
                  host_positions: bool = False):
    """Config ``number`` (2-5) with its positions generated on the GPU: a dict
    with ``x, y, z`` (fp32 cuda tensors), ``mass`` / ``h0`` (numpy fp64), K,
    box; ``pos`` (numpy (n, 3) fp64 of the fp32 values) when
    ``host_positions``.  ``n_ranks > 1`` is the weak-scaled set (n_ranks x
    particles, halos and volume)."""
    seed = number if seed is None else seed
    n, box, n_halos, k, conc, x_max = _config_table(number, n_ranks)
    if number == 5:
        n_bg = int(round(0.05 * n))
        start = np.array([0, n - n_bg], dtype=np.int64)
        halo = np.array([[0.5 * box, 0.5 * box, 0.5 * box, 1.0, 1.0]])
    else:
        start, halo = halo_table(n, box, n_halos, seed)
    x, y, z = nfw_device(n, box, start, halo, seed, conc, x_max, device=device)
    w = dict(x=x, y=y, z=z, mass=np.full(n, 1.0 / n), h0=np.full(n, _initial_h(box, n, k)), k=k, box=box,
             periodic=True, fp32=True, halo_start=start, halo=halo, seed=seed, concentration=conc, x_max=x_max,
             name=f"C{number} device-generated {n} fp32")
    if host_positions:
        w["pos"] = np.stack([t.cpu().numpy() for t in (x, y, z)], axis=1).astype(np.float64)
    return w


def config_weak(number: int, n_ranks: int, seed: int | None = None):
    """Weak-scaled form of config ``number`` for ``n_ranks`` GPUs: n_ranks
    times the particles, halos and volume (box side x n_ranks^(1/3)) of the
    one-GPU config, the same generator; n_ranks = 1 is ``config(number)``."""
    if n_ranks == 1 or number not in (2, 3, 6):
        return config(number, seed)
    seed = number if seed is None else seed
    g = n_ranks ** (1.0 / 3.0)
    if number in (2, 3):
        n1, box1, halos1 = {2: (1 << 20, 100.0, 200), 3: (1 << 24, 100.0 * 16 ** (1.0 / 3.0), 20000)}[number]
        n, box = n1 * n_ranks, box1 * g
        pos, vel, _ = nfw_halos(n, box, halos1 * n_ranks, seed)
    else:
        n, box = (1 << 20) * n_ranks, 100.0 * g
        pos = (np.random.default_rng(seed).random((n, 3)) * box).astype(np.float32).astype(np.float64)
        pos[pos >= box] = np.float64(np.nextafter(np.float32(box), np.float32(0.0)))
        vel = np.zeros((n, 3), np.float32)
    return dict(pos=pos, vel=vel, mass=np.full(n, 1.0 / n), h0=np.full(n, _initial_h(box, n, 64)), k=64, box=box,
                periodic=True, fp32=True, name=f"C{number} weak x{n_ranks}: {n} fp32")


def _initial_h(box: float, n: int, k: int) -> float:
    # density.py:136-140
    return box * (3.0 * k / (4.0 * math.pi * n)) ** (1.0 / 3.0)
