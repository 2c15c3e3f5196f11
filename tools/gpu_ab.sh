# A/B of env settings on the bench (C2 and optionally C3): bash tools/gpu_ab.sh "ENV1" "ENV2" ...
cd $GRAFT_REPO_ROOT
CFGS=${AB_CFGS:-2}
for e in "$@"; do for c in $CFGS; do
  env $e timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/ab.json 2> /tmp/ab.err
  python -c "
import json
d=json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1]); print('$e', 'C$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()}, 'tests', d.get('pair_tests_per_step'), 'known_ms', d.get('known_ms_per_step'))
" 2>&1 | tail -1
done; done
