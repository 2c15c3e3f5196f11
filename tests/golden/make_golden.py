"""Generate the golden vectors that pin the oracle (and through it the GPU).

Runs the REFERENCE implementation itself (``sphlab`` from
/root/reference/pkg/src, read-only) on seeded inputs and stores inputs and
outputs as small .npz fixtures next to this script.  Run it in the build
container (the reference does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Each fixture records the reference call it came from.  Positions are stored
verbatim except for the uniform-box cases, which store the seed and an FNV-1a
digest of the positions (the repo regenerates them bit-exactly, see
paper_1612_06090_b200/workload.py and tests/test_workload.py).
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

import sphlab  # noqa: E402
from sphlab import (  # noqa: E402
    WorkloadKind, WorkloadSpec, build_octree, compute_density_pass, density_checksum,
    generate, new_particle_array, preset_config, range_query, QueryWorkspace,
)
from sphlab.snapshot import checksum64  # noqa: E402

THREADS = os.cpu_count() or 1


def fnv(arr) -> str:
    return f"{checksum64(np.ascontiguousarray(arr).tobytes()):016x}"


def run_pass(p, k, preset="optimised", max_iterations=100):
    work = p.copy()
    rho, st = compute_density_pass(work, preset_config(preset, k_neighbors=k),
                                   thread_count=THREADS, max_iterations=max_iterations)
    return work, rho, st


def pack_particles(p):
    return dict(x=np.asarray(p["x"]), y=np.asarray(p["y"]), z=np.asarray(p["z"]),
                mass=np.asarray(p["mass"]), h0=np.asarray(p["smoothing_length"]))


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def full_case(name, p, k, note, **extra):
    work, rho, st = run_pass(p, k)
    tree = build_octree((np.asarray(p["x"]), np.asarray(p["y"]), np.asarray(p["z"])))
    save(name, **pack_particles(p), k=k, h=np.asarray(work["smoothing_length"]), rho=rho,
         todo=st.todo_sizes, perm=tree.particle_perm, checksum=density_checksum(rho),
         note=note, **extra)


def uniform_case(name, n, seed, k, box=1.0, h0=None, mass=None, sample=2048):
    p = generate(WorkloadSpec(WorkloadKind.UNIFORM_BOX, n, box_side=box, seed=seed),
                 k_neighbors=k)
    if mass is not None:
        p["mass"] = mass
    if h0 is not None:
        p["smoothing_length"] = h0
    pos_digest = fnv(np.column_stack([p["x"], p["y"], p["z"]]))
    work, rho, st = run_pass(p, k)
    h = np.asarray(work["smoothing_length"])
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(n, size=min(sample, n), replace=False))
    tree = build_octree((np.asarray(p["x"]), np.asarray(p["y"]), np.asarray(p["z"])))
    save(name, n=n, seed=seed, k=k, box=box,
         h0=np.float64(p["smoothing_length"][0]), mass=np.float64(p["mass"][0]),
         pos_digest=pos_digest, sample_idx=idx, sample_h=h[idx], sample_rho=rho[idx],
         h_digest=fnv(h), rho_checksum=density_checksum(rho), todo=st.todo_sizes,
         perm_digest=fnv(tree.particle_perm.astype("<i8")),
         first_pos=np.column_stack([p["x"][:8], p["y"][:8], p["z"][:8]]),
         note=f"generate(UNIFORM_BOX, {n}, box={box}, seed={seed}, k={k}); "
              f"compute_density_pass optimised, {THREADS} threads")


def main():
    # Config 1 of BASELINE.json (open boundary, the reference's semantics):
    # 32,768 uniform, m = 1/N, h0 = 2 * N^(-1/3), K = 64.
    n1 = 32768
    uniform_case("c1_uniform32k", n1, seed=1, k=64, h0=2.0 * n1 ** (-1.0 / 3.0), mass=1.0 / n1)
    # the reference's own 4096-particle smoke run (reference h0 rule)
    uniform_case("uniform4096_seed81", 4096, seed=81, k=64, sample=4096)

    # clustered (test_density.py:159-166 shape, larger), positions stored
    p = generate(WorkloadSpec(WorkloadKind.GAUSSIAN_BLOBS, 3000, seed=7, blob_count=3),
                 k_neighbors=12)
    full_case("blobs3000_k12", p, 12, "generate(GAUSSIAN_BLOBS, 3000, seed=7, blobs=3), K=12")
    p = generate(WorkloadSpec(WorkloadKind.GAUSSIAN_BLOBS, 4000, seed=5, blob_count=6,
                              blob_sigma=0.02), k_neighbors=48)
    full_case("blobs4000_k48", p, 48, "generate(GAUSSIAN_BLOBS, 4000, seed=5, blobs=6, sigma=0.02), K=48")

    # lattice: every particle has distance ties at its K-th neighbour
    p = generate(WorkloadSpec(WorkloadKind.LATTICE, 16 ** 3), k_neighbors=32)
    full_case("lattice4096_k32", p, 32, "generate(LATTICE, 4096), K=32")

    # K+1 particle cluster with unequal masses (test_density.py:141-156 shape)
    k = 32
    rng = np.random.default_rng(1)
    p = new_particle_array(k + 1)
    p["id"] = np.arange(k + 1)
    for f, v in zip("xyz", rng.random((3, k + 1)) * 0.01 + 0.5):
        p[f] = v
    p["mass"] = rng.random(k + 1) + 0.5
    p["smoothing_length"] = 1.0
    full_case("cluster33_k32", p, k, "K+1 cluster, unequal masses, h0 = 1")

    # fp32-representable positions in a box of side 100 (the fp32 configs'
    # contract: the reference sees the fp32 values widened to fp64)
    rng = np.random.default_rng(2)
    n = 6000
    p = new_particle_array(n)
    pos = (rng.random((n, 3)) * 100.0).astype(np.float32).astype(np.float64)
    # a dense clump to add density contrast
    pos[:1500] = (50.0 + rng.normal(0.0, 1.5, (1500, 3))).astype(np.float32).astype(np.float64)
    p["x"], p["y"], p["z"] = pos[:, 0], pos[:, 1], pos[:, 2]
    p["mass"] = (rng.random(n) + 0.5).astype(np.float32).astype(np.float64)
    p["smoothing_length"] = sphlab.initial_smoothing_length(100.0, n, 64)
    full_case("f32pos6000_k64", p, 64, "fp32-representable positions, box 100, clump, K=64")

    # perm fixtures with coincident clusters (octree.py:75-86 guard)
    rng = np.random.default_rng(3)
    pos = rng.random((3000, 3))
    pos[100:120] = pos[5]          # 21 coincident (> leaf capacity)
    pos[200:206] = pos[7]          # 7 coincident
    pos[300:340] = [0.5, 0.5, 0.5]  # 40 coincident at the root centre
    tree = build_octree(pos)
    save("perm_coincident3000", x=pos[:, 0], y=pos[:, 1], z=pos[:, 2], perm=tree.particle_perm,
         n_nodes=tree.n_nodes, note="uniform 3000 + coincident groups of 21, 7, 40")
    # clustered perm
    p = generate(WorkloadSpec(WorkloadKind.GAUSSIAN_BLOBS, 8000, seed=11, blob_count=5,
                              blob_sigma=0.01), k_neighbors=64)
    tree = build_octree((np.asarray(p["x"]), np.asarray(p["y"]), np.asarray(p["z"])))
    save("perm_blobs8000", x=np.asarray(p["x"]), y=np.asarray(p["y"]), z=np.asarray(p["z"]),
         perm=tree.particle_perm.astype(np.int32), n_nodes=tree.n_nodes,
         note="generate(GAUSSIAN_BLOBS, 8000, seed=11, blobs=5, sigma=0.01)")

    # fixed-h neighbour counts (octree range_query with exclude = self)
    p = generate(WorkloadSpec(WorkloadKind.UNIFORM_BOX, 4096, seed=81), k_neighbors=64)
    x, y, z = (np.asarray(p[f]) for f in "xyz")
    rng = np.random.default_rng(4)
    h = p["smoothing_length"] * rng.uniform(0.3, 2.0, 4096)
    # a few radii exactly at a pair distance (inclusive boundary)
    tree = build_octree((x, y, z))
    for i in range(0, 64):
        j = (i * 37 + 11) % 4096
        d2 = ((x[j] - x[i]) * (x[j] - x[i]) + (y[j] - y[i]) * (y[j] - y[i])) + (z[j] - z[i]) * (z[j] - z[i])
        h[i] = math.sqrt(d2)
    ws = QueryWorkspace()
    cnt = np.array([range_query(tree, (x[i], y[i], z[i]), h[i], ws, exclude=i)[0].size
                    for i in range(4096)], dtype=np.int32)
    save("counts4096", h=h, counts=cnt, seed=81, note="range_query(tree, pos_i, h_i, exclude=i).size "
         "on generate(UNIFORM_BOX, 4096, seed=81) positions")

    # periodic box via image augmentation (reference run on originals + images)
    n, box, k = 2048, 1.0, 32
    p = generate(WorkloadSpec(WorkloadKind.UNIFORM_BOX, n, seed=9), k_neighbors=k)
    x, y, z = (np.asarray(p[f]) for f in "xyz")
    margin = 0.3
    xs, ys, zs = [x], [y], [z]
    for sx in (-1, 0, 1):
        for sy in (-1, 0, 1):
            for sz in (-1, 0, 1):
                if sx == sy == sz == 0:
                    continue
                ix, iy, iz = x + sx * box, y + sy * box, z + sz * box
                keep = ((ix >= -margin) & (ix < box + margin) & (iy >= -margin) &
                        (iy < box + margin) & (iz >= -margin) & (iz < box + margin))
                xs.append(ix[keep]); ys.append(iy[keep]); zs.append(iz[keep])
    ax, ay, az = np.concatenate(xs), np.concatenate(ys), np.concatenate(zs)
    q = new_particle_array(ax.shape[0])
    q["x"], q["y"], q["z"] = ax, ay, az
    q["mass"] = 1.0
    q["smoothing_length"] = p["smoothing_length"][0]
    work, rho, _ = run_pass(q, k)
    hmax = float(np.max(work["smoothing_length"][:n]))
    assert hmax < margin, hmax
    save("periodic2048_k32", x=x, y=y, z=z, box=box, k=k, h0=np.float64(p["smoothing_length"][0]),
         h=np.asarray(work["smoothing_length"][:n]), rho=rho[:n], margin=margin,
         note="reference on originals + periodic images within 0.3 of the unit box")

    # error behaviour
    errs = {}
    p = generate(WorkloadSpec(WorkloadKind.UNIFORM_BOX, 16, seed=2), k_neighbors=8)
    try:
        compute_density_pass(p.copy(), preset_config("optimised", k_neighbors=32), max_iterations=5)
    except sphlab.ConvergenceError as e:
        errs["convergence"] = str(e)
    p = new_particle_array(40)
    rng = np.random.default_rng(4)
    for f in "xyz":
        p[f] = rng.random(40)
        p[f][:6] = 0.25
    p["mass"] = 1.0
    p["smoothing_length"] = 0.3
    try:
        compute_density_pass(p.copy(), preset_config("optimised", k_neighbors=4))
    except sphlab.DegenerateWorkloadError as e:
        errs["degenerate"] = str(e)
    save("errors", convergence=errs["convergence"], degenerate=errs["degenerate"],
         deg_x=np.asarray(p["x"]), deg_y=np.asarray(p["y"]), deg_z=np.asarray(p["z"]))
    # constants
    save("constants", h_growth=sphlab.H_GROWTH, norm=sphlab.WENDLAND_C6_NORM,
         w_samples_r=np.linspace(0, 1.2, 13), w_samples=sphlab.kernel_w(np.linspace(0, 1.2, 13), 1.1))


if __name__ == "__main__":
    main()
