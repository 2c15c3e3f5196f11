# usage: bash tools/knob_sweep.sh -- A/B of env-var knobs on the bench (one GPU)
run() { python bench.py --config $1 --steps ${STEPS:-15} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$2', 'c$1', round(d['ms_per_step'],3))"; }
for r in 1 2 3; do
 for c in 1 2 3 5; do
  run $c base; SPH_SEEDM=1.08 run $c seedm1.08
 done
done
