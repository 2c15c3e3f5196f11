# GPU tests, bench C3 + C2, launch list C3
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/rNN_pytest.log 2>&1; tail -3 gpurun_out/rNN_pytest.log
timeout 900 python bench.py > gpurun_out/rNN_bench_c3.json 2> gpurun_out/rNN_bench_c3.err; echo bench_rc=$?
timeout 600 python bench.py --config 2 > gpurun_out/rNN_bench_c2.json 2> gpurun_out/rNN_bench_c2.err; echo bench2_rc=$?
python -c "
import json
for c in (3,2):
    d=json.loads(open('gpurun_out/rNN_bench_c%d.json'%c).read().strip().splitlines()[-1]); print(c, d['ms_per_step'], d['value'], d['e2e']['value'], d['kernel_ms_per_step'], d['roofline']['frac'])
"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rNN_c3_launches.csv \
  python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/rNN_ncu_list.log 2>&1; echo list_rc=$?
python tools/launches.py gpurun_out/rNN_c3_launches.csv 40 2>&1 | tail -32
