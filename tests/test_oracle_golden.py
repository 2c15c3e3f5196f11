"""Pins the CPU oracle against vectors produced by the reference itself.

The fixtures come from tests/golden/make_golden.py (which imports the
reference sphlab package); every comparison here is bit-exact.
"""
import numpy as np
import pytest

import oracle
from conftest import golden
from paper_1612_06090_b200 import workload
from paper_1612_06090_b200.checksum import array_digest, density_checksum


def _uniform_inputs(g):
    n, seed, box = int(g["n"]), int(g["seed"]), float(g["box"])
    pos = workload.uniform_box(n, seed, box)
    assert array_digest(pos) == str(g["pos_digest"])
    assert np.array_equal(pos[:8], g["first_pos"])
    return pos


@pytest.mark.parametrize("name", ["c1_uniform32k", "uniform4096_seed81"])
def test_uniform_cases_bit_exact(name):
    g = golden(name)
    pos = _uniform_inputs(g)
    n = pos.shape[0]
    res = oracle.density_pass(pos[:, 0], pos[:, 1], pos[:, 2], np.full(n, float(g["mass"])),
                              np.full(n, float(g["h0"])), int(g["k"]))
    assert np.array_equal(res.todo_sizes, g["todo"])
    idx = g["sample_idx"]
    assert np.array_equal(res.h[idx], g["sample_h"])
    assert np.array_equal(res.rho[idx], g["sample_rho"])
    assert array_digest(res.h) == str(g["h_digest"])
    assert density_checksum(res.rho) == str(g["rho_checksum"])
    assert not res.flags.any()
    assert array_digest(oracle.perm(pos[:, 0], pos[:, 1], pos[:, 2]).astype("<i8")) == str(g["perm_digest"])


@pytest.mark.parametrize("name", ["blobs3000_k12", "blobs4000_k48", "lattice4096_k32",
                                  "cluster33_k32", "f32pos6000_k64"])
@pytest.mark.parametrize("threads", [1, 0])
def test_full_cases_bit_exact(name, threads):
    g = golden(name)
    res = oracle.density_pass(g["x"], g["y"], g["z"], g["mass"], g["h0"], int(g["k"]),
                              threads=threads)
    assert np.array_equal(res.h, g["h"])
    assert np.array_equal(res.rho, g["rho"])
    assert np.array_equal(res.todo_sizes, g["todo"])
    assert density_checksum(res.rho) == str(g["checksum"])
    assert np.array_equal(oracle.perm(g["x"], g["y"], g["z"]), g["perm"])


@pytest.mark.parametrize("name", ["perm_coincident3000", "perm_blobs8000"])
def test_perm_bit_exact(name):
    g = golden(name)
    assert np.array_equal(oracle.perm(g["x"], g["y"], g["z"]), g["perm"].astype(np.int64))


def test_fixed_h_counts_bit_exact():
    g = golden("counts4096")
    pos = workload.uniform_box(4096, int(g["seed"]))
    got = oracle.counts(pos[:, 0], pos[:, 1], pos[:, 2], g["h"])
    assert np.array_equal(got, g["counts"])


def test_periodic_images_bit_exact():
    g = golden("periodic2048_k32")
    n = g["x"].shape[0]
    res = oracle.density_pass_periodic(g["x"], g["y"], g["z"], np.ones(n), np.full(n, float(g["h0"])),
                                       int(g["k"]), float(g["box"]), margin=float(g["margin"]))
    assert np.array_equal(res.h, g["h"])
    assert np.array_equal(res.rho, g["rho"])


def test_error_messages_match_reference():
    g = golden("errors")
    pos = workload.uniform_box(16, 2)
    h0 = np.full(16, (3.0 * 8 / (4.0 * np.pi * 16)) ** (1.0 / 3.0))
    with pytest.raises(oracle.OracleConvergenceError) as e:
        oracle.density_pass(pos[:, 0], pos[:, 1], pos[:, 2], np.ones(16), h0, 32, max_iterations=5)
    assert str(e.value) == str(g["convergence"])
    with pytest.raises(oracle.OracleDegenerateError) as e:
        oracle.density_pass(g["deg_x"], g["deg_y"], g["deg_z"], np.ones(40), np.full(40, 0.3), 4)
    assert str(e.value) == str(g["degenerate"])


def test_constants():
    g = golden("constants")
    assert oracle.H_GROWTH == float(g["h_growth"])
    assert oracle.WENDLAND_C6_NORM == float(g["norm"])
    for r, w in zip(g["w_samples_r"], g["w_samples"]):
        assert oracle.kernel_w(r, 1.1) == w


def test_brute_force_agrees_with_oracle():
    g = golden("blobs3000_k12")
    h, rho = oracle.brute_force(g["x"], g["y"], g["z"], g["mass"], 12)
    assert np.array_equal(h, g["h"])
    assert np.allclose(rho, g["rho"], rtol=1e-12, atol=0)
