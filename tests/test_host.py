"""CPU-only tests: the C ABI library loads and exports every declared symbol,
and the host-side mirror of the reference API behaves like the reference
(constants, presets, validation, layouts, checksums, workload streams)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle
import paper_1612_06090_b200 as sph
from conftest import ROOT, golden
from paper_1612_06090_b200 import _lib, workload
from paper_1612_06090_b200.checksum import FNV_OFFSET_BASIS, density_checksum, fnv1a64


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "sph_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sph_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared_functions()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED_SYMBOLS)


def test_library_loads_without_gpu_and_refuses_compute():
    lib = _lib.load()
    if lib.sph_device_count() == 0:
        with pytest.raises(RuntimeError, match="no CUDA device"):
            _lib.context(0)


def test_struct_layouts():
    assert ctypes.sizeof(_lib.SphParams) == 48
    assert _lib.SphStats.todo_sizes.offset == 8


def test_fnv_known_answers():
    # test_snapshot.py:35-38 of the reference
    assert fnv1a64(b"") == FNV_OFFSET_BASIS == 0xCBF29CE484222325
    assert fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert density_checksum(np.array([], dtype=np.float64)) == "cbf29ce484222325"


def test_splitmix_known_answer_and_uniform_stream():
    # test_workload.py:27-30 of the reference: splitmix64(seed 0) first output
    from paper_1612_06090_b200.workload import _splitmix_values
    assert int(_splitmix_values(0, 0, 1)[0]) == 0xE220A8397B1DCDAF
    g = golden("uniform4096_seed81")
    pos = workload.uniform_box(4096, 81)
    assert np.array_equal(pos[:8], g["first_pos"])


def test_constants_and_presets():
    g = golden("constants")
    assert sph.H_GROWTH == float(g["h_growth"])
    assert sph.WENDLAND_C6_NORM == float(g["norm"])
    assert abs(sph.WENDLAND_C6_NORM - 6.78895304126366) < 1e-13
    assert sph.DEFAULT_K == 295 and sph.DEFAULT_MAX_ITERATIONS == 100
    assert set(sph.PRESETS) == {"original", "todo-list", "lockless", "soa", "vectorised", "optimised"}
    cfg = sph.preset_config("optimised", k_neighbors=32, chunk_size=4)
    assert cfg.k_neighbors == 32 and cfg.chunk_size == 4
    with pytest.raises(ValueError, match="unknown preset"):
        sph.preset_config("fastest")
    with pytest.raises(ValueError):
        sph.preset_config("optimised", k_neighbors=0)


def test_kernel_w_matches_reference_samples():
    g = golden("constants")
    got = sph.kernel_w(g["w_samples_r"], 1.1)
    assert np.array_equal(got, g["w_samples"])
    assert sph.kernel_w(0.0, 1.0) == sph.WENDLAND_C6_NORM
    with pytest.raises(ValueError):
        sph.kernel_w(0.5, 0.0)
    with pytest.raises(ValueError):
        sph.kernel_w(-0.1, 1.0)
    # M4 extension: normalised to one over R^3
    r = np.linspace(0, 1, 200001)
    w = sph.kernel_w(r, 1.0, sph.KernelKind.M4)
    assert abs(np.trapezoid(4 * math.pi * r * r * w, r) - 1.0) < 1e-6


def test_smoothing_length_helpers():
    h0 = sph.initial_smoothing_length(1.0, 4096, 64)
    assert np.isclose(4096 * (4.0 / 3.0) * math.pi * h0 ** 3, 64.0)
    with pytest.raises(ValueError):
        sph.initial_smoothing_length(0.0, 10, 3)
    assert sph.adjust_smoothing_length(1.0, 5, 8) == (sph.H_GROWTH, True)
    assert sph.adjust_smoothing_length(1.0, 8, 8, 0.7) == (0.7, False)
    with pytest.raises(ValueError):
        sph.adjust_smoothing_length(1.0, 8, 8)
    with pytest.raises(ValueError):
        sph.adjust_smoothing_length(1.0, -1, 8)


def test_density_interact_matches_oracle_kernel():
    masses = np.array([2.0, 3.0, 5.0])
    d2 = np.array([0.04, 0.25, 4.0])
    idx = np.array([2, 0, 1])
    want = 5.0 * oracle.kernel_w(0.2, 1.0) + 2.0 * oracle.kernel_w(0.5, 1.0)
    for style in sph.LoopStyle:
        assert np.isclose(sph.density_interact(masses, 1.0, d2, idx, style), want, rtol=1e-15)
    assert sph.density_interact(masses, 1.0, np.array([]), np.array([], dtype=np.int64)) == 0.0


def test_record_layout():
    dt = sph.aos_dtype()
    assert dt.itemsize == 224 and sph.LIVE_RECORD_BYTES == 57
    offs = {name: dt.fields[name][1] for name in dt.names if name != "pad"}
    assert offs == {"id": 0, "x": 8, "y": 16, "z": 24, "mass": 32, "smoothing_length": 40, "density": 48,
                    "needs_recompute": 56}
    assert sph.aos_dtype(64).itemsize == 64
    with pytest.raises(ValueError):
        sph.aos_dtype(32)
    p = sph.new_particle_array(5)
    p["x"] = np.arange(5)
    soa = sph.gather_to_soa(p)
    soa.density[:] = 7.0
    sph.scatter_from_soa(soa, p)
    assert np.all(p["density"] == 7.0)
    with pytest.raises(ValueError):
        sph.scatter_from_soa(soa, p, {"bogus"})


def test_validation_before_any_device_work():
    cfg = sph.preset_config("optimised", k_neighbors=4)
    with pytest.raises(ValueError):
        sph.compute_density_pass(sph.new_particle_array(0), cfg)
    with pytest.raises(ValueError):
        sph.compute_density_pass(sph.new_particle_array(8), cfg, thread_count=0)


def test_nfw_generator_shape_and_rules():
    pos, vel, counts = workload.nfw_halos(20000, 100.0, 30, seed=4)
    assert pos.shape == (20000, 3) and vel.shape == (20000, 3)
    assert counts.sum() == 16000  # 80% in halos, largest-remainder rounding
    assert pos.min() >= 0.0 and pos.max() < 100.0
    assert np.array_equal(pos.astype(np.float32).astype(np.float64), pos)  # fp32-representable
    w = workload.config(1)
    assert w["pos"].shape == (32768, 3) and w["h0"][0] == 2.0 * 32768 ** (-1.0 / 3.0)


def test_bench_reference_arm_json_contract():
    # bench.py --impl reference (the CPU port of the reference pass) prints one
    # JSON line with the driver's keys; tiny sample so it runs in seconds
    import json
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "1", "--warmup", "0", "--cpu-seconds", "1"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert "workload" in line["config"]
