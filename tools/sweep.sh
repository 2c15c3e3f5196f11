for cfg in 6 1 2; do
  timeout 300 python bench.py --config $cfg --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>gpurun_out/sw.err || tail -5 gpurun_out/sw.err
  python -c "
import json; d=json.load(open('gpurun_out/sw.json'))
print('config $cfg', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, d['pair_tests_per_step'], d['search_rounds'], d['select_rounds'], 'eff', d['search_efficiency'])"
done
