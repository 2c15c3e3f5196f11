"""The reference's own command line (`sphlab gen / run / report / verify`,
reference cli.py) with `sphlab.bench.compute_density_pass` routed to the B200
pass (sphlab_adapter.install, the seam of reference bench.py:25-30, 144):

    python tools/sphlab_gpu.py run workload.sphk --variant optimised --save-results gpu.sphk

The reference package is imported from baseline/_ref (offline install that
travels with the repo) or, in the build container, /root/reference/pkg/src."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for cand in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "sphlab")):
        sys.path.insert(0, cand)
        break
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import sphlab  # noqa: E402
import sphlab.cli  # noqa: E402

from paper_1612_06090_b200 import sphlab_adapter  # noqa: E402


def main(argv):
    sphlab_adapter.install(sphlab)
    return sphlab.cli.main(argv)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
