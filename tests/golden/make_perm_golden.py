"""Golden particle orders for leaf capacities other than 8 and for trees
deeper than the 21 levels of a 63-bit key: the reference's own
build_octree(positions, leaf_capacity).particle_perm (octree.py:306-348,
MAX_TREE_DEPTH = 48), run here in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_perm_golden.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from sphlab import WorkloadKind, WorkloadSpec, build_octree, generate  # noqa: E402


def main():
    p = generate(WorkloadSpec(WorkloadKind.GAUSSIAN_BLOBS, 5000, seed=23), k_neighbors=32)
    x, y, z = (np.ascontiguousarray(p[f]) for f in "xyz")
    caps = np.array([1, 3, 16, 32])
    perms = np.stack([build_octree((x, y, z), leaf_capacity=int(c)).particle_perm for c in caps])
    # deep trees: tight clusters far below 2^-21 of the root extent (unit box)
    rng = np.random.default_rng(8)
    base = rng.random((3000, 3))
    clusters = []
    for c, (m, s) in enumerate([(12, 1e-9), (20, 3e-10), (31, 1e-11), (9, 4e-8), (40, 2e-9)]):
        ctr = rng.random(3)
        pts = ctr + s * rng.standard_normal((m, 3))
        if c == 4:
            pts[10:20] = pts[10]  # coincident points inside a deep cluster (non-separable leaf)
        clusters.append(pts)
    dpos = np.concatenate([base] + clusters)
    order = rng.permutation(dpos.shape[0])
    dpos = np.ascontiguousarray(dpos[order])
    dx, dy, dz = (np.ascontiguousarray(dpos[:, i]) for i in range(3))
    deep8 = build_octree((dx, dy, dz)).particle_perm
    deep4 = build_octree((dx, dy, dz), leaf_capacity=4).particle_perm
    path = os.path.join(HERE, "perm_caps_deep.npz")
    np.savez_compressed(path, x=x, y=y, z=z, caps=caps, perms=perms.astype(np.int32), dx=dx, dy=dy, dz=dz,
                        deep8=deep8.astype(np.int32), deep4=deep4.astype(np.int32),
                        note="build_octree(..., leaf_capacity).particle_perm on generate(GAUSSIAN_BLOBS, 5000, "
                             "seed=23) and on 3000 uniform points + 5 clusters of 9-40 points at 1e-11..4e-8")
    print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main()
