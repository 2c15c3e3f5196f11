# usage: bash tools/knob_sweep.sh -- A/B of env-var knobs on the bench (one GPU)
run() { python bench.py --config $1 --steps ${STEPS:-15} --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$2', 'c$1', round(d['ms_per_step'],3))"; }
for r in 1 2; do
 for c in 1 3; do
  run $c base; SPH_SEED=12 run $c seed12; SPH_SEED=16 run $c seed16
 done
 SPH_SEED=16 SPH_SEEDM=1.05 run 5 s16m1.05; SPH_SEED=16 SPH_SEEDM=1.05 run 2 s16m1.05
done
