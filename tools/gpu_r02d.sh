# r02d: the per-cell group kernel: fallback counters, GPU tests, bench C2/C3 (G = 8, 4; per-target known kernel for A/B)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
SPH_DEBUG=1 timeout 300 python -c "
import numpy as np, paper_1612_06090_b200 as sph
from paper_1612_06090_b200 import workload
for c in (2,5):
    w = workload.config_device(c, host_positions=True); p=w['pos'].astype(np.float32)
    h,rho,fl,st = sph.density_pass_soa(p[:,0],p[:,1],p[:,2],w['mass'],w['h0'],w['k'],periodic=True,box=w['box'])
    print(c, st.device['t_known_ms'], st.device['known_fallbacks'], st.device['t_kernel_ms'])
" > gpurun_out/dbg.log 2>&1
tail -12 gpurun_out/dbg.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
tail -5 gpurun_out/pytest.log
for v in "2 8" "2 4" "1 8"; do set -- $v; for c in 2 3; do
SPH_KNOWN=$1 SPH_GROUP_G=$2 timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_k$1g$2_c$c.json 2> gpurun_out/ab_k$1g$2_c$c.err
python -c "
import json
d=json.loads(open('gpurun_out/ab_k$1g$2_c$c.json').read().strip().splitlines()[-1]); print('known=$1 g=$2 c=$c', d['ms_per_step'], d['kernel_ms_per_step'], d['roofline']['frac'])
"
done; done
