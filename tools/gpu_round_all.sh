# Round artefacts on one GPU (run under gpurun): default bench (C3), reference arm, C1/C2/C4/C5 bench lines,
# ncu launch list of C3, full ncu captures of the C3 search launches.  usage: bash tools/gpu_round_all.sh TAG
cd $GRAFT_REPO_ROOT
TAG=${1:-rXX}
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/${TAG}_bench_c3_default.json 2> gpurun_out/${TAG}_bench_c3.err; echo "bench rc=$? $(( $(date +%s) - t0 ))s"
t0=$(date +%s); timeout 1500 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_c3.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$? $(( $(date +%s) - t0 ))s"
for c in 1 2 5 4; do
  timeout 1500 python bench.py --config $c > gpurun_out/${TAG}_bench_c${c}_all.json 2> gpurun_out/${TAG}_bench_c${c}.err; echo "bench c$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c3_launches.csv \
  python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
bash tools/gpu_ncu_c3.sh $TAG
python - <<PY
import json,glob
for f in sorted(glob.glob('gpurun_out/${TAG}_bench_*.json')):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), (d.get('roofline') or {}).get('frac'), (d.get('cpu_baseline') or {}).get('value'))
    except Exception as e: print(f, 'ERR', e)
PY
