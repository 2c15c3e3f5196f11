"""Randomised parity sweep (run on a GPU box): seeded random particle sets
(uniform, Gaussian blobs, NFW halos, coincident clumps), random N, K, box,
precision and boundary, each against the CPU oracle (h bit-exact, density
rel 1e-12 fp64 / 1e-4 fp32, todo trace exact).

    python tools/fuzz.py [cases] [seed]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1612_06090_b200 as sph  # noqa: E402
from paper_1612_06090_b200 import workload  # noqa: E402


def make(rng):
    kind = rng.choice(["uniform", "blobs", "nfw", "clumps", "coincident"])
    n = int(rng.integers(300, 40000))
    k = int(rng.choice([1, 2, 5, 16, 32, 64, 64, 64, 100, 128, 200]))
    k = min(k, max(1, n - 2)) if rng.random() < 0.97 else n + 5  # K unreachable now and then
    periodic = bool(rng.random() < 0.5)
    box = float(rng.choice([1.0, 10.0, 100.0]))
    if kind == "uniform":
        pos = rng.random((n, 3)) * box
    elif kind == "blobs":
        nb = int(rng.integers(1, 8))
        c = rng.random((nb, 3)) * box
        pos = c[rng.integers(0, nb, n)] + rng.normal(0.0, box * rng.uniform(0.005, 0.05), (n, 3))
    elif kind == "nfw":
        pos, _, _ = workload.nfw_halos(n, box, int(rng.integers(1, 30)), seed=int(rng.integers(1 << 30)))
    elif kind == "coincident":  # exact duplicates: the K-th may sit at zero distance
        base = rng.random((max(2, n // int(rng.integers(2, 200))), 3)) * box
        pos = base[rng.integers(0, len(base), n)]
    else:  # clumps of near-coincident points plus background
        m = n // 2
        c = rng.random((max(1, m // 40), 3)) * box
        pos = np.concatenate([c[rng.integers(0, len(c), m)] + rng.normal(0.0, box * 1e-4, (m, 3)),
                              rng.random((n - m, 3)) * box])
    pos = np.mod(pos, box)
    f32 = bool(rng.random() < 0.6)
    if f32:
        pos = pos.astype(np.float32).astype(np.float64)
        pos[pos >= box] = np.float64(np.nextafter(np.float32(box), np.float32(0.0)))
    mass = rng.random(n) + 0.5
    h0 = np.full(n, sph.initial_smoothing_length(box, n, k) * rng.uniform(0.3, 3.0))
    return kind, pos, mass, h0, k, periodic, box, f32


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
    bad = 0
    t0 = time.time()
    for c in range(cases):
        kind, pos, mass, h0, k, periodic, box, f32 = make(rng)
        n = len(pos)
        arr = pos.astype(np.float32) if f32 else pos
        try:
            if periodic:
                want = oracle.density_pass_periodic(pos[:, 0], pos[:, 1], pos[:, 2], mass, h0, k, box)
            else:
                want = oracle.density_pass(pos[:, 0], pos[:, 1], pos[:, 2], mass, h0, k)
            werr = None
        except Exception as e:  # the reference raises: the GPU must raise the same kind
            want, werr = None, type(e).__name__
        try:
            h, rho, _, st = sph.density_pass_soa(arr[:, 0], arr[:, 1], arr[:, 2], mass, h0, k, periodic=periodic,
                                                 box=box)
            gerr = None
        except Exception as e:
            gerr = type(e).__name__
        if werr or gerr:
            ok = (werr is not None) == (gerr is not None)
            msg = f"errors oracle={werr} gpu={gerr}"
        else:
            rel = float(np.max(np.abs(rho - want.rho) / want.rho))
            tol = 1e-4 if f32 else 1e-12
            ok = np.array_equal(h, want.h) and rel <= tol and np.array_equal(st.todo_sizes, want.todo_sizes)
            msg = f"h_mis={int(np.sum(h != want.h))} rho_rel={rel:.1e} todo_ok={np.array_equal(st.todo_sizes, want.todo_sizes)}"
        bad += not ok
        print(f"{c:3d} {'ok ' if ok else 'BAD'} {kind:7s} n={n:6d} k={k:3d} periodic={periodic!s:5s} box={box:5.0f} "
              f"f32={f32!s:5s} {msg}", flush=True)
    print(f"{cases - bad}/{cases} ok in {time.time() - t0:.0f}s")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
