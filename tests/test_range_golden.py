"""The range-query golden vectors (tests/golden/make_rq_golden.py: the
reference's range_query around arbitrary centres, octree.py:351-379) pinned
against an unfused fp64 brute force restatement of the same predicate."""
import numpy as np

from conftest import golden


def brute(x, y, z, c, r, ex):
    dx, dy, dz = x - c[0], y - c[1], z - c[2]
    d2 = (dx * dx + dy * dy) + dz * dz  # numpy: each op rounded, no contraction
    sel = np.nonzero(d2 <= r * r)[0]
    sel = sel[sel != ex]
    return sel, d2[sel]


def test_golden_range_queries_match_brute_force():
    g = golden("rq_points")
    x, y, z = g["x"], g["y"], g["z"]
    off = g["offsets"]
    assert off[-1] == g["idx"].size
    for q in range(g["radii"].size):
        idx, d2 = brute(x, y, z, g["centers"][q], g["radii"][q], g["exclude"][q])
        assert np.array_equal(idx, g["idx"][off[q]:off[q + 1]]), q
        assert np.array_equal(d2, g["d2"][off[q]:off[q + 1]]), q
