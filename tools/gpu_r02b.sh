# r02b: the known-radius kernel: GPU tests, bench C2/C3, debug counters
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
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
tail -5 gpurun_out/pytest.log
for c in 2 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
python -c "
import json
for c in (2,3):
    d=json.loads(open('gpurun_out/bench_c%d.json'%c).read().strip().splitlines()[-1]); print(c, d['ms_per_step'], d['value'], d['e2e']['value'], d['kernel_ms_per_step'], d['roofline']['frac'])
"
