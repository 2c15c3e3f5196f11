"""particle_perm on the GPU for leaf capacities 1-32 and for trees deeper
than the 21 levels of a 63-bit key (runs of identical keys subdivided down to
MAX_TREE_DEPTH = 48, octree.py:31, 36-176), bit-exact against the reference's
own orders (tests/golden/perm_caps_deep.npz); the density pass over the deep
set against the oracle."""
import numpy as np
import pytest

import oracle
from conftest import golden
from paper_1612_06090_b200 import density as gd
from paper_1612_06090_b200 import octree

pytestmark = pytest.mark.gpu


def test_perm_leaf_capacities_match_reference():
    g = golden("perm_caps_deep")
    for c, want in zip(g["caps"], g["perms"]):
        assert np.array_equal(octree.particle_perm((g["x"], g["y"], g["z"]), leaf_capacity=int(c)), want), c


def test_perm_deep_trees_match_reference():
    g = golden("perm_caps_deep")
    pos = (g["dx"], g["dy"], g["dz"])
    assert np.array_equal(octree.particle_perm(pos), g["deep8"])
    assert np.array_equal(octree.particle_perm(pos, leaf_capacity=4), g["deep4"])


def test_density_pass_over_deep_tree_matches_oracle():
    g = golden("perm_caps_deep")
    x, y, z = g["dx"], g["dy"], g["dz"]
    n, k = x.shape[0], 16  # > the 10 coincident points of one cluster
    m = np.full(n, 1.0 / n)
    h0 = np.full(n, 0.05)
    h, rho, fl, st = gd.density_pass_soa(x, y, z, m, h0, k)
    ref = oracle.density_pass(x, y, z, m, h0, k)
    assert np.array_equal(h, ref.h)
    np.testing.assert_allclose(rho, ref.rho, rtol=1e-12, atol=0)
    assert list(st.todo_sizes) == list(ref.todo_sizes)


def test_more_than_32_distinct_points_in_one_key_cell():
    # 40 distinct positions within 1e-10: one search cell of 40 particles
    rng = np.random.default_rng(2)
    pos = np.concatenate([rng.random((500, 3)), 0.5 + 1e-10 * rng.standard_normal((40, 3))])
    x, y, z = (np.ascontiguousarray(pos[:, i]) for i in range(3))
    assert np.array_equal(octree.particle_perm((x, y, z)), oracle.perm(x, y, z))
    m, h0 = np.ones(540), np.full(540, 0.1)
    h, rho, _, _ = gd.density_pass_soa(x, y, z, m, h0, 8)
    ref = oracle.density_pass(x, y, z, m, h0, 8)
    assert np.array_equal(h, ref.h)
    np.testing.assert_allclose(rho, ref.rho, rtol=1e-12, atol=0)
