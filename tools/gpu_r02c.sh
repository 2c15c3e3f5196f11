# r02c: A/B the known-radius kernel against the general kernel alone; launch list with it on
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for kn in 0 1; do for c in 2 3; do
SPH_KNOWN=$kn timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_k${kn}_c$c.json 2> gpurun_out/ab_k${kn}_c$c.err
python -c "
import json
d=json.loads(open('gpurun_out/ab_k${kn}_c$c.json').read().strip().splitlines()[-1]); print('known=$kn c=$c', d['ms_per_step'], d['kernel_ms_per_step'], d['roofline']['frac'])
"
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_c2_launches.csv \
  python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c_ncu_list.log 2>&1; echo list_rc=$?
python tools/launches.py gpurun_out/r02c_c2_launches.csv 40 2>&1 | tail -60
