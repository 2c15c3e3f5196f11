"""The cropped periodic oracle (oracle.periodic_crop) used by the full-size
GPU tests gives exactly the full periodic oracle's answer for the targets."""
import numpy as np

import oracle
from paper_1612_06090_b200 import workload


def test_periodic_crop_matches_full_oracle():
    n, box, k = 20000, 40.0, 16
    pos, _, _ = workload.nfw_halos(n, box, 30, seed=5, halo_fraction=0.5)
    x, y, z = pos[:, 0], pos[:, 1], pos[:, 2]
    mass = np.full(n, 1.0 / n)
    h0 = np.full(n, workload._initial_h(box, n, k))
    full = oracle.density_pass_periodic(x, y, z, mass, h0, k, box)
    tg = np.sort(np.random.default_rng(1).choice(n, size=40, replace=False))
    margin = 1.05 * float(full.h[tg].max())
    sel = oracle.periodic_crop(x, y, z, box, tg, margin)
    assert sel.size < n
    loc = np.searchsorted(sel, tg)
    h0c = h0[sel].copy()
    h0c[loc] = full.h[tg] * 1.01
    got = oracle.density_pass_periodic(x[sel], y[sel], z[sel], mass[sel], h0c, k, box, margin=margin, targets=loc)
    assert np.array_equal(got.h[loc], full.h[tg])
    assert np.allclose(got.rho[loc], full.rho[tg], rtol=1e-13, atol=0)
