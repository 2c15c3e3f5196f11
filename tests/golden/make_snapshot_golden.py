"""Golden SPHK snapshot written by the REFERENCE (sphlab, /root/reference,
read-only), the way `sphlab gen` writes one (cli.py:117-142): a "meta" JSON
section and a "particles" section (snapshot.encode_particles), plus the
reference's own pass on the decoded particles.  Run in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_snapshot_golden.py
"""
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF)

from sphlab import WorkloadKind, WorkloadSpec, compute_density_pass, generate, preset_config, snapshot  # noqa: E402


def main():
    spec = WorkloadSpec(kind=WorkloadKind.UNIFORM_BOX, n_particles=3000, box_side=1.0, seed=17)
    p = generate(spec, k_neighbors=32)
    meta = {"format": "sphlab-workload", "kind": spec.kind.value, "n_particles": spec.n_particles,
            "box_side": spec.box_side, "seed": spec.seed, "blob_count": spec.blob_count,
            "blob_sigma": spec.blob_sigma, "k_neighbors": 32, "record_bytes": 224}
    path = os.path.join(HERE, "snap_uniform3000_k32.sphk")
    snapshot.dump(path, {"meta": json.dumps(meta, sort_keys=True).encode("utf-8"),
                         "particles": snapshot.encode_particles(p)})
    back = snapshot.decode_particles(snapshot.load(path)["particles"])
    rho, st = compute_density_pass(back, preset_config("optimised", k_neighbors=32))
    np.savez_compressed(os.path.join(HERE, "snap_uniform3000_k32.npz"), h=np.asarray(back["smoothing_length"]),
                        rho=rho, todo=st.todo_sizes,
                        particles_checksum=f"{snapshot.checksum64(snapshot.load(path)['particles']):016x}",
                        note="sphlab.snapshot.dump of generate(UNIFORM_BOX, 3000, seed=17, k=32); pass: "
                             "compute_density_pass(decoded, preset optimised, K=32)")
    print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main()
