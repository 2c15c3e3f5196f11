"""Golden vectors for range queries around arbitrary centres: the reference's
own range_query(tree, center, radius, workspace, exclude) (octree.py:351-379)
on a clustered set, run here in the build container (the reference does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_rq_golden.py

Each query's (index, d2) list is stored sorted by index (the reference lists
the same set in tree order)."""
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from sphlab import QueryWorkspace, WorkloadKind, WorkloadSpec, build_octree, generate, range_query  # noqa: E402


def main():
    p = generate(WorkloadSpec(WorkloadKind.GAUSSIAN_BLOBS, 3000, seed=17), k_neighbors=32)
    x, y, z = (np.ascontiguousarray(p[f]) for f in "xyz")
    n = x.shape[0]
    tree = build_octree((x, y, z))
    rng = np.random.default_rng(3)
    lo = np.array([x.min(), y.min(), z.min()])
    hi = np.array([x.max(), y.max(), z.max()])
    ext = hi - lo
    cen, rad, exc = [], [], []
    for q in range(40):  # at particles, half of them excluding themselves
        i = int(rng.integers(n))
        cen.append((x[i], y[i], z[i]))
        rad.append(float(rng.uniform(0.005, 0.08)))
        exc.append(i if q % 2 == 0 else -1)
    for q in range(30):  # anywhere in (and around) the box
        cen.append(tuple(lo - 0.2 * ext + rng.random(3) * 1.4 * ext))
        rad.append(float(rng.uniform(0.0, 0.25)))
        exc.append(-1)
    for q in range(10):  # radius exactly a pair distance (inclusive boundary), and zero radius
        i, j = int(rng.integers(n)), int(rng.integers(n))
        d2 = ((x[j] - x[i]) * (x[j] - x[i]) + (y[j] - y[i]) * (y[j] - y[i])) + (z[j] - z[i]) * (z[j] - z[i])
        cen.append((x[i], y[i], z[i]))
        rad.append(math.sqrt(d2) if q < 7 else 0.0)
        exc.append(-1)
    ws = QueryWorkspace()
    offs, idxs, d2s = [0], [], []
    for c, r, e in zip(cen, rad, exc):
        idx, d2 = range_query(tree, c, r, ws, exclude=e)
        o = np.argsort(idx, kind="stable")
        idxs.append(np.array(idx[o], dtype=np.int64))
        d2s.append(np.array(d2[o], dtype=np.float64))
        offs.append(offs[-1] + idx.size)
    path = os.path.join(HERE, "rq_points.npz")
    np.savez_compressed(path, x=x, y=y, z=z, centers=np.array(cen, dtype=np.float64), radii=np.array(rad),
                        exclude=np.array(exc, dtype=np.int64), offsets=np.array(offs, dtype=np.int64),
                        idx=np.concatenate(idxs), d2=np.concatenate(d2s),
                        note="range_query(build_octree(generate(GAUSSIAN_BLOBS, 3000, seed=17)), c, r, ws, exclude)")
    print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main()
