# usage: bash tools/knob_sweep.sh -- A/B of env-var knobs on the bench (one GPU)
run() { python bench.py --config $1 --steps ${STEPS:-15} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$2', 'c$1', round(d['ms_per_step'],3))"; }
for r in 1 2; do
 for c in 2 5; do
  run $c base
  SPH_NEARF=0.4 run $c nearf0.4; SPH_NEARF=0.6 run $c nearf0.6
  SPH_TLISTCAP=3 run $c tcap3; SPH_TLISTCAP=5 run $c tcap5
  SPH_SEEDM=1.08 run $c seedm1.08; SPH_SEEDM=1.13 run $c seedm1.13
 done
done
