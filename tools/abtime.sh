# usage: bash tools/abtime.sh CONFIG REPS  -- alternates every _variants/*.so, 20-step bench each, prints ms
for r in $(seq 1 ${2:-2}); do
  for lib in _variants/*.so; do
    cp "$lib" paper_1612_06090_b200/libsph_b200.so
    python bench.py --config ${1:-2} --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', round(d['ms_per_step'],3))"
  done
done
