"""Every pipeline of the library against the CPU oracle.

The default pass: seeds (every 12th sorted target) through the general
per-target kernel, then the lane kernel (sph_lane.cu: bundles of 32 sorted
neighbours, one lane per target) and, for what it leaves, neighbour-cell
lists and the per-target kernel (SPH_KNOWN=0: the per-target kernel for every
non-seed target).  The fallbacks (the per-target kernel for what the lane
kernel leaves, the collect instance for overflowed neighbour lists, the
walking select/density kernels) only run on a few targets of large inputs, so
they are forced here with margins and list capacities.  Each configuration
runs in a fresh process because the switches are read when the library
context is created.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

CONFIGS = {
    "default": {},
    "per_target_only": {"SPH_KNOWN": "0"},
    "lane_tight_margin": {"SPH_LANEM": "1.0"},                      # many lanes with < K within R: per-target kernel
    "lane_wide_margin_short_lists": {"SPH_LANEM": "1.8", "SPH_LANE_LEXTRA": "8"},   # full lists, crowded brackets
    "lane_short_streams": {"SPH_LANE_STREAM": "600"},              # most bundles bail to the per-target kernel
    "lane_no_exclusion": {"SPH_LANEX": "0"},
    "lane_from_dense_seeds": {"SPH_LANE_NOSEED": "0"},
    "lane_low_quantile": {"SPH_LANE_CALQ": "0.3"},                  # most lanes with < K within R
    "lane_high_quantile_sparse_sample": {"SPH_LANE_CALQ": "0.99", "SPH_LANE_CAL": "2048"},
    "cell_lists_far_records": {"SPH_KNOWN": "0", "SPH_NEARF": "0.3"},
    "lane_then_cell_lists_far_records": {"SPH_NEARF": "0.3"},
    "per_target_small_lists": {"SPH_KNOWN": "0", "SPH_TLISTCAP": "1"},
    "lane_then_small_lists": {"SPH_TLISTCAP": "1", "SPH_LANE_STREAM": "900"},
    "per_target_seed_stride_8": {"SPH_KNOWN": "0", "SPH_SEED": "8"},
    "lane_seed_stride_8": {"SPH_SEED": "8"},
    "per_target_crowded_brackets": {"SPH_KNOWN": "0", "SPH_TLISTCAP": "1", "SPH_CCAP": "48"},
    "per_target_unseeded_no_cell_lists": {"SPH_SEED": "0", "SPH_CLIST": "0"},
}


@pytest.mark.parametrize("cfg", sorted(CONFIGS))
def test_pipeline_matches_oracle(cfg):
    env = dict(os.environ)
    env.update(CONFIGS[cfg])
    r = subprocess.run([sys.executable, os.path.join(HERE, "_path_worker.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    for name, v in res.items():
        assert v["h_exact"], (cfg, name)
        assert v["todo_exact"], (cfg, name)
        tol = 1e-4 if "_f32_" in name else 1e-12
        assert v["rho_rel"] <= tol, (cfg, name, v["rho_rel"])
