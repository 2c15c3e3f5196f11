# one debug pass per env setting on C2 (and C5 when SWEEP_C5=1): bash tools/gpu_sweep_env.sh "A=1 B=2" "A=3" ...
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1 PYTHONPATH=$GRAFT_REPO_ROOT
cat > /tmp/sweep_one.py <<'PY'
import os, sys, numpy as np, paper_1612_06090_b200 as sph
from paper_1612_06090_b200 import workload
cfgs = [int(c) for c in os.environ.get("SWEEP_CFGS", "2").split(",")]
for c in cfgs:
    w = workload.config_device(c, host_positions=True); p = w['pos'].astype(np.float32)
    ts = []
    for rep in range(3):
        h, rho, fl, st = sph.density_pass_soa(p[:,0],p[:,1],p[:,2],w['mass'],w['h0'],w['k'],periodic=True,box=w['box'])
        ts.append(st.device['t_known_ms'])
    print(sys.argv[1], 'C%d' % c, 'known_ms %.3f' % min(ts), 'kernel', {k: round(v, 3) for k, v in st.device['t_kernel_ms'].items()}, 'fb', st.device['known_fallbacks'], 'tests', st.device.get('pair_tests'), flush=True)
PY
for e in "$@"; do
  env $e SPH_DEBUG=1 timeout 300 python /tmp/sweep_one.py "$e" 2>&1 | grep -v "^\[sph collect\]\|^\[sph warp\]" | tail -2
done
