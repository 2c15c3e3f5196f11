"""Run every golden density fixture through the library and report mismatches (debug aid)."""
import glob, sys
import numpy as np
sys.path.insert(0, ".")
from paper_1612_06090_b200.density import density_pass_soa

for f in sorted(glob.glob("tests/golden/*.npz")):
    d = np.load(f)
    if "h" not in d.files or "x" not in d.files:
        continue
    k = int(d["k"]) if "k" in d.files else 64
    kw = {}
    if "mass" not in d.files:
        continue
    try:
        h, rho, fl, st = density_pass_soa(d["x"], d["y"], d["z"], d["mass"], d["h0"], k, **kw)
        print(f, "max rel h", float(np.max(np.abs(h - d["h"]) / d["h"])), "rho", float(np.max(np.abs(rho - d["rho"]) / d["rho"])))
    except Exception as e:
        print(f, "ERROR", e)
