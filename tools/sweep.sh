for cfg in "2.0" "3.0"; do
 for c in 2 6; do
  SPH_SUBD_RETRY=$cfg timeout 120 python bench.py --config $c --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>gpurun_out/sw.err || tail -5 gpurun_out/sw.err
  python -c "
import json; d=json.load(open('gpurun_out/sw.json'))
print('retry $cfg config $c', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items()}, d['pair_tests_per_step'], d['search_rounds'])"
 done
done
