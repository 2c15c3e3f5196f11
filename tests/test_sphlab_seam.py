"""The reference harness through the repo's pass: with the
reference package importable (this build container; absent on the GPU box,
where the test skips), `sphlab_adapter.install` routes
`sphlab.bench.run_benchmark` through the repo's `compute_density_pass`.  With
no GPU here, the CPU oracle stands in for the device behind the same
signature; the harness' records and checksum must equal the reference's own
run, and the reference's exception types must surface."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


@pytest.fixture(scope="module")
def sphlab():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    import sphlab as s
    return s


def _oracle_pass(particles, config, thread_count=1, max_iterations=100):
    # the repo's compute_density_pass contract, computed by the CPU oracle
    import oracle
    from paper_1612_06090_b200 import density as gd
    k = config.k_neighbors
    try:
        r = oracle.density_pass(np.array(particles["x"]), np.array(particles["y"]), np.array(particles["z"]),
                                np.array(particles["mass"]), np.array(particles["smoothing_length"]), k,
                                max_iterations)
    except oracle.OracleConvergenceError as e:
        raise gd.ConvergenceError(str(e))
    except oracle.OracleDegenerateError as e:
        raise gd.DegenerateWorkloadError(str(e))
    particles["smoothing_length"] = r.h
    particles["density"] = r.rho
    particles["needs_recompute"] = 0
    todo = np.asarray(r.todo_sizes, dtype=np.int64)
    st = gd.PassStats(iteration_count=len(todo), todo_sizes=todo,
                      phase_times={"tree_build": 0.0, "search": 0.0, "select": 0.0, "interact": 0.0, "layout": 0.0},
                      contention_time=0.0, items_per_worker=todo.reshape(-1, 1), skipped_items=0, t_total=0.0)
    return np.array(r.rho), st


def test_run_benchmark_through_the_seam(sphlab):
    from paper_1612_06090_b200 import sphlab_adapter
    spec = sphlab.WorkloadSpec(kind=sphlab.WorkloadKind.UNIFORM_BOX, n_particles=3000, box_side=1.0, seed=9)
    p = sphlab.generate(spec, k_neighbors=32)
    cfg = sphlab.preset_config("optimised", k_neighbors=32)
    want, _ = sphlab.bench.run_benchmark(p, cfg, "optimised", 1, 1)
    undo = sphlab_adapter.install(sphlab, gpu_pass=_oracle_pass)
    try:
        assert sphlab.bench.compute_density_pass is not sphlab.density.compute_density_pass
        got, rho = sphlab.bench.run_benchmark(p, cfg, "optimised", 1, 2)
    finally:
        undo()
    assert sphlab.bench.compute_density_pass is sphlab.density.compute_density_pass
    assert got[0].checksum_hex == want[0].checksum_hex == got[1].checksum_hex
    assert got[0].iterations == want[0].iterations


def test_reference_exception_types_surface(sphlab):
    from paper_1612_06090_b200 import sphlab_adapter
    p = sphlab.new_particle_array(20)
    rng = np.random.default_rng(1)
    for f in "xyz":
        p[f] = rng.random(20)
    p["mass"] = 1.0
    p["smoothing_length"] = 0.1
    run = sphlab_adapter.make_pass(sphlab, gpu_pass=_oracle_pass)
    with pytest.raises(sphlab.ConvergenceError):
        run(p.copy(), sphlab.preset_config("optimised", k_neighbors=32))
