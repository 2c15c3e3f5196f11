"""One density pass of a bench config with the library's debug output (set SPH_DEBUG=1)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1612_06090_b200 import workload
from paper_1612_06090_b200.density import density_pass_soa

c = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = workload.config(c)
dt = np.float32 if w["fp32"] else np.float64
p = w["pos"].astype(dt)
m = w["mass"].astype(dt)
for rep in range(2):
    t = time.time()
    h, rho, fl, st = density_pass_soa(p[:, 0], p[:, 1], p[:, 2], m, w["h0"], w["k"], periodic=w["periodic"], box=w["box"])
    print("pass", rep, time.time() - t, st.todo_sizes.tolist(), file=sys.stderr)
np.save("gpurun_out/h_c%d.npy" % c, h)
