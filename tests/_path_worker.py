"""Worker for tests/test_gpu_paths.py: runs the pass on a few seeded inputs in a
fresh process (the pipeline selection is read from SPH_* environment
variables when the library context is created) and checks every result
against the CPU oracle.  Prints one JSON line."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_1612_06090_b200 as sph  # noqa: E402
from paper_1612_06090_b200 import workload  # noqa: E402


def cases():
    rng = np.random.default_rng(7)
    n = 30000
    pos = np.concatenate([rng.normal(10.0 + 8 * b, 0.6, (n // 5, 3)) for b in range(5)])
    yield "blobs_f32_k64", np.abs(pos).astype(np.float32), rng.random(n) + 0.5, 64, None
    # fp64 positions that are fp32 values: fp32 search, fp64 term-for-term densities
    yield "blobs_auto_k48", np.abs(pos).astype(np.float32).astype(np.float64), rng.random(n) + 0.5, 48, None
    pos, _ = workload.single_halo(20000, 4.0, 23)
    yield "halo_f32_k128", pos.astype(np.float32), np.ones(20000), 128, None
    pos, _, _ = workload.nfw_halos(12000, 10.0, 20, seed=5)
    yield "nfw_periodic_f32_k64", pos.astype(np.float32), np.ones(12000), 64, 10.0
    pos = workload.uniform_box(8000, 3, 1.0)
    yield "uniform_periodic_f64_k32", pos, np.full(8000, 1.0 / 8000), 32, 1.0


def main():
    out = {}
    for name, pos, mass, k, box in cases():
        p64 = pos.astype(np.float64)
        n = len(p64)
        h0 = np.full(n, sph.initial_smoothing_length(box or float(p64.max()), n, k))
        if box:
            want = oracle.density_pass_periodic(p64[:, 0], p64[:, 1], p64[:, 2], mass, h0, k, box)
            h, rho, _, st = sph.density_pass_soa(pos[:, 0], pos[:, 1], pos[:, 2], mass, h0, k, periodic=True, box=box)
        else:
            want = oracle.density_pass(p64[:, 0], p64[:, 1], p64[:, 2], mass, h0, k)
            prec = "auto" if "_auto_" in name else None
            h, rho, _, st = sph.density_pass_soa(pos[:, 0], pos[:, 1], pos[:, 2], mass, h0, k, precision=prec)
        out[name] = {"h_exact": bool(np.array_equal(h, want.h)),
                     "rho_rel": float(np.max(np.abs(rho - want.rho) / want.rho)),
                     "todo_exact": bool(np.array_equal(st.todo_sizes, want.todo_sizes))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
