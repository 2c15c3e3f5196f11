"""The device tree object and its query around arbitrary centres
(octree.build_octree / range_query / range_query_many -> C ABI
sph_octree_build / sph_octree_query) against the reference's own
range_query outputs (tests/golden/rq_points.npz), bit-exact: same index set,
same fp64 squared distances, inclusive boundary, exclude, zero radius,
centres outside the particle box."""
import numpy as np
import pytest

from conftest import golden
from paper_1612_06090_b200 import octree

pytestmark = pytest.mark.gpu


def test_range_query_many_matches_reference_golden():
    g = golden("rq_points")
    tree = octree.build_octree((g["x"], g["y"], g["z"]))
    off, idx, d2 = octree.range_query_many(tree, g["centers"], g["radii"], g["exclude"])
    assert np.array_equal(off, g["offsets"])
    assert np.array_equal(idx, g["idx"])
    assert np.array_equal(d2, g["d2"])


def test_single_queries_and_errors():
    g = golden("rq_points")
    tree = octree.build_octree(np.stack([g["x"], g["y"], g["z"]], axis=1))
    off = g["offsets"]
    for q in (0, 1, 45, 72, 79):
        idx, d2 = octree.range_query(tree, g["centers"][q], float(g["radii"][q]), exclude=int(g["exclude"][q]))
        assert np.array_equal(idx, g["idx"][off[q]:off[q + 1]])
        assert np.array_equal(d2, g["d2"][off[q]:off[q + 1]])
    with pytest.raises(ValueError, match="non-negative"):
        octree.range_query(tree, (0.5, 0.5, 0.5), -1.0)
    assert np.array_equal(tree.particle_perm, octree.particle_perm((g["x"], g["y"], g["z"])))


def test_large_batch_grows_the_output():
    rng = np.random.default_rng(1)
    pos = rng.random((50000, 3)).astype(np.float32)
    tree = octree.build_octree(pos)
    cen = rng.random((300, 3))
    rad = np.full(300, 0.08)
    off, idx, d2 = octree.range_query_many(tree, cen, rad)
    x, y, z = (pos[:, i].astype(np.float64) for i in range(3))
    for q in range(0, 300, 37):
        dx, dy, dz = x - cen[q, 0], y - cen[q, 1], z - cen[q, 2]
        dd = (dx * dx + dy * dy) + dz * dz
        want = np.nonzero(dd <= rad[q] * rad[q])[0]
        assert np.array_equal(idx[off[q]:off[q + 1]], want)
        assert np.array_equal(d2[off[q]:off[q + 1]], dd[want])
