"""The reference's own command line on the GPU: `sphlab gen`
writes a workload file, `sphlab run` runs it on the CPU (the reference) and,
through tools/sphlab_gpu.py (the reference CLI with sphlab_adapter.install),
on the B200; `sphlab verify --rtol 1e-12` accepts the GPU densities against
the reference's, the iteration counts printed by both runs agree, and
`sphlab report` builds its speedup table from the GPU rows (reference
cli.py:145-277)."""
import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "sphlab")),
                                 reason="reference package not installed in baseline/_ref")]

ENV = dict(os.environ, NUMBA_CACHE_DIR="/tmp/numba_cache")


def ref_cli(*args):
    code = "import sys; sys.path.insert(0, %r); import sphlab.cli; sys.exit(sphlab.cli.main(sys.argv[1:]))" % REF
    return subprocess.run([sys.executable, "-c", code, *args], capture_output=True, text=True, env=ENV, timeout=900)


def gpu_cli(*args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sphlab_gpu.py"), *args],
                          capture_output=True, text=True, env=ENV, timeout=900)


@pytest.mark.parametrize("kind", ["uniform", "blobs"])
def test_sphlab_gen_run_verify_report_on_the_gpu(tmp_path, kind):
    wl = str(tmp_path / "wl.sphk")
    r = ref_cli("gen", "--kind", kind, "--n", "20000", "--seed", "5", "--k", "64", "--out", wl)
    assert r.returncode == 0, r.stderr
    ref_out, gpu_out = str(tmp_path / "ref.sphk"), str(tmp_path / "gpu.sphk")
    r = ref_cli("run", wl, "--variant", "optimised", "--threads", "4", "--csv", str(tmp_path / "ref.csv"),
                "--save-results", ref_out)
    assert r.returncode == 0, r.stderr
    g = gpu_cli("run", wl, "--variant", "optimised", "--repeats", "2", "--csv", str(tmp_path / "gpu.csv"),
                "--save-results", gpu_out)
    assert g.returncode == 0, g.stderr
    it_ref = re.findall(r"iterations=(\d+)", r.stdout)
    it_gpu = re.findall(r"iterations=(\d+)", g.stdout)
    assert it_ref and it_gpu == it_ref * 2
    v = ref_cli("verify", ref_out, gpu_out, "--rtol", "1e-12")
    assert v.returncode == 0, v.stdout + v.stderr
    # the report's baseline row (variant original, 1 thread) from the GPU too
    g2 = gpu_cli("run", wl, "--variant", "original", "--threads", "1", "--csv", str(tmp_path / "gpu.csv"))
    assert g2.returncode == 0, g2.stderr
    rep = ref_cli("report", str(tmp_path / "gpu.csv"))
    assert rep.returncode == 0, rep.stderr
    assert "optimised" in rep.stdout
