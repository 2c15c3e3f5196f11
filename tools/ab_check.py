"""A/B check of two library settings on one bench config (run on a GPU box):
h must be bit-identical, density within rel 1e-5 (fp32 sums); prints timings.

    python tools/ab_check.py CONFIG "ENV_A" "ENV_B"      e.g. 2 "SPH_BUNDLE=0" "SPH_BUNDLE=1"
"""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, time, json
import numpy as np
sys.path.insert(0, %r)
from paper_1612_06090_b200 import workload
from paper_1612_06090_b200.density import density_pass_soa
c = int(sys.argv[1]); out = sys.argv[2]
w = workload.config(c)
dt = np.float32 if w["fp32"] else np.float64
p = w["pos"].astype(dt)
ts = []
for rep in range(4):
    t = time.time()
    h, rho, fl, st = density_pass_soa(p[:, 0], p[:, 1], p[:, 2], w["mass"], w["h0"], w["k"], periodic=w["periodic"], box=w["box"])
    ts.append(time.time() - t)
np.savez(out, h=h, rho=rho)
print(json.dumps({"t_ms": [round(x * 1e3, 2) for x in ts], "todo": st.todo_sizes.tolist()[:6],
                  "device": {k: v for k, v in st.device.items() if k in ("pair_tests", "accepted_pairs", "gpu_launches", "t_kernel_ms", "t_stage_ms")}}))
""" % ROOT


def run(cfg, setting, out):
    env = dict(os.environ)
    for kv in setting.split():
        k, v = kv.split("=", 1)
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD, str(cfg), out], env=env, capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        print(r.stdout[-2000:], r.stderr[-4000:])
        raise SystemExit(f"{setting}: rc {r.returncode}")
    sys.stderr.write(r.stderr[-3000:])
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    cfg = int(sys.argv[1])
    sa, sb = sys.argv[2], sys.argv[3]
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    fa = os.path.join(ROOT, "gpurun_out", f"ab_a_{cfg}.npz")
    fb = os.path.join(ROOT, "gpurun_out", f"ab_b_{cfg}.npz")
    ra = run(cfg, sa, fa)
    rb = run(cfg, sb, fb)
    A, B = np.load(fa), np.load(fb)
    hd = int(np.sum(A["h"] != B["h"]))
    rel = float(np.max(np.abs(A["rho"] - B["rho"]) / np.maximum(np.abs(A["rho"]), 1e-300)))
    print(f"config {cfg}: [{sa}] {ra}\n          [{sb}] {rb}\n  h mismatches {hd} of {A['h'].size}, rho max rel {rel:.3e}")
    if hd:
        i = np.nonzero(A["h"] != B["h"])[0][:10]
        print("  first mismatches", i.tolist(), A["h"][i].tolist(), B["h"][i].tolist())
    return 0 if hd == 0 and rel < 1e-5 else 1


if __name__ == "__main__":
    sys.exit(main())
