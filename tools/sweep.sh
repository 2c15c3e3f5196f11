# usage: bash tools/sweep.sh "ENV1=a ENV2=b" "ENV1=c" ...   (each arg one setting, run on configs 6 and 2)
for setting in "$@"; do
 for c in 6 2; do
  env $setting timeout 120 python bench.py --config $c --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>gpurun_out/sw.err || tail -5 gpurun_out/sw.err
  python -c "
import json; d=json.load(open('gpurun_out/sw.json'))
print('$setting | config $c', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, d['pair_tests_per_step'], d['search_rounds'], d['select_rounds'])"
 done
done
