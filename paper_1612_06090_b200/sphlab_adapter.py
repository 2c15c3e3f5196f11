"""Route the reference harness (`sphlab run / report / verify`) through the GPU.

`sphlab.bench.run_benchmark` looks `compute_density_pass` up in the
`sphlab.bench` namespace at call time (reference bench.py:25-30, 144; the seam
its own test_bench.py:150-168 patches).  `install(sphlab)` puts the GPU pass
there, translating this package's exceptions into the reference's own
`ConvergenceError` / `DegenerateWorkloadError` (which `sphlab`'s CLI catches,
cli.py:294-295) and its `PassStats` into the reference's dataclass, so the
harness' CSV rows, checksums and nondeterminism check run unchanged.

    import sphlab
    from paper_1612_06090_b200 import sphlab_adapter
    undo = sphlab_adapter.install(sphlab)      # ... sphlab.bench.run_benchmark(...) now runs on the GPU
    undo()
"""

from __future__ import annotations

from . import density as _gpu


def make_pass(sphlab, gpu_pass=None):
    """The reference-typed pass: (particles, config, thread_count,
    max_iterations) -> (densities, sphlab PassStats)."""
    ref = sphlab.density
    run = gpu_pass or _gpu.compute_density_pass

    def compute_density_pass(particles, config, thread_count=1, max_iterations=ref.DEFAULT_MAX_ITERATIONS):
        try:
            rho, st = run(particles, config, thread_count, max_iterations)
        except _gpu.ConvergenceError as exc:
            raise ref.ConvergenceError(str(exc)) from exc
        except _gpu.DegenerateWorkloadError as exc:
            raise ref.DegenerateWorkloadError(str(exc)) from exc
        stats = ref.PassStats(iteration_count=st.iteration_count, todo_sizes=st.todo_sizes,
                              phase_times=dict(st.phase_times), contention_time=st.contention_time,
                              items_per_worker=st.items_per_worker, skipped_items=st.skipped_items,
                              t_total=st.t_total)
        return rho, stats

    return compute_density_pass


def install(sphlab, gpu_pass=None):
    """Patch `sphlab.bench.compute_density_pass`; returns a function that
    restores the original."""
    prev = sphlab.bench.compute_density_pass
    sphlab.bench.compute_density_pass = make_pass(sphlab, gpu_pass)

    def undo():
        sphlab.bench.compute_density_pass = prev

    return undo
