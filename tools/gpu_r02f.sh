# r02f: per-cell group kernel with walk + retries: fallback counters, GPU tests, bench C2/C3 (G = 4, 8)
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for g in 4 8; do
SPH_GROUP_G=$g SPH_DEBUG=1 timeout 300 python -c "
import numpy as np, paper_1612_06090_b200 as sph
from paper_1612_06090_b200 import workload
for c in (2,5):
    w = workload.config_device(c, host_positions=True); p=w['pos'].astype(np.float32)
    h,rho,fl,st = sph.density_pass_soa(p[:,0],p[:,1],p[:,2],w['mass'],w['h0'],w['k'],periodic=True,box=w['box'])
    print('G=$g', c, st.device['t_known_ms'], st.device['known_fallbacks'], st.device['t_kernel_ms'])
" > gpurun_out/dbg_g$g.log 2>&1
grep -v "^\[sph collect\]" gpurun_out/dbg_g$g.log | tail -8
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
tail -15 gpurun_out/pytest.log
for g in 4 8; do for c in 2 3; do
SPH_GROUP_G=$g timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_g${g}_c$c.json 2> gpurun_out/ab_g${g}_c$c.err
python -c "
import json
d=json.loads(open('gpurun_out/ab_g${g}_c$c.json').read().strip().splitlines()[-1]); print('g=$g c=$c', d['ms_per_step'], d['kernel_ms_per_step'], d['roofline']['frac'], d['pair_tests_per_step'])
"
done; done
