"""The oracle's particle_perm for leaf capacities 1-32 and trees deeper than
21 levels (depth up to 48) against the reference's own orders
(tests/golden/perm_caps_deep.npz, make_perm_golden.py)."""
import numpy as np

import oracle
from conftest import golden


def test_oracle_perm_leaf_capacities():
    g = golden("perm_caps_deep")
    for c, want in zip(g["caps"], g["perms"]):
        assert np.array_equal(oracle.perm(g["x"], g["y"], g["z"], leaf_capacity=int(c)), want), c


def test_oracle_perm_deep_trees():
    g = golden("perm_caps_deep")
    assert np.array_equal(oracle.perm(g["dx"], g["dy"], g["dz"]), g["deep8"])
    assert np.array_equal(oracle.perm(g["dx"], g["dy"], g["dz"], leaf_capacity=4), g["deep4"])
