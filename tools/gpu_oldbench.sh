# bench C2 at old commits built under _variants/<tag> (git worktrees) vs the current tree
cd $GRAFT_REPO_ROOT
for d in r02a; do
  (cd _variants/$d && timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['ms_per_step'], d['kernel_ms_per_step'])")
done
for kn in 0 1 2 3; do SPH_KNOWN=$kn SPH_GROUP_G=4 SPH_GROUP_R0F=1.15 timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('now known=$kn', d['ms_per_step'], d['kernel_ms_per_step'])"; done
