import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1612_06090_b200 as sph
rng = np.random.default_rng(1)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
pos = (rng.random((n, 3)) * 10).astype(np.float32)
h, rho, fl, st = sph.density_pass_soa(pos[:, 0], pos[:, 1], pos[:, 2], np.ones(n), 0.5, 32)
print("ok", h[:3], st.device["t_kernel_ms"])
