# bench lines for every config on one B200 (C4: 134M particles on one GPU)
cd $GRAFT_REPO_ROOT
for c in 1 2 5 4; do
  st=10; [ $c = 4 ] && st=5
  timeout 1500 python bench.py --config $c --steps $st --warmup 3 > gpurun_out/r02o_bench_c$c.json 2> gpurun_out/r02o_bench_c$c.err; echo "c$c rc=$?"
  python -c "
import json
d=json.loads(open('gpurun_out/r02o_bench_c$c.json').read().strip().splitlines()[-1]); print($c, round(d['ms_per_step'],3), '%.3e'%d['value'], '%.3e'%d['e2e']['value'], (d.get('cpu_baseline') or {}).get('value'))
"
done
