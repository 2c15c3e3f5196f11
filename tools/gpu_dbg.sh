# debug counters of the pass on C2 and C5: bash tools/gpu_dbg.sh TAG
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
SPH_DEBUG=1 timeout 300 python -c "
import numpy as np, paper_1612_06090_b200 as sph
from paper_1612_06090_b200 import workload
for c in (2,5):
    w = workload.config_device(c, host_positions=True); p=w['pos'].astype(np.float32)
    for rep in range(2):
        h,rho,fl,st = sph.density_pass_soa(p[:,0],p[:,1],p[:,2],w['mass'],w['h0'],w['k'],periodic=True,box=w['box'])
    print('C%d'%c, 'known_ms', st.device['t_known_ms'], 'fallbacks', st.device['known_fallbacks'], st.device['t_kernel_ms'], 'tests', st.device.get('pair_tests'))
" > gpurun_out/dbg_$1.log 2>&1
grep -v "^\[sph collect\]" gpurun_out/dbg_$1.log | tail -12
