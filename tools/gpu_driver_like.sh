# what the driver runs at round end (one B200): smoke, default bench, default reference arm, with wall times
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
t0=$(date +%s); timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/drv_smoke.log 2>&1; echo "smoke rc=$? $(( $(date +%s) - t0 ))s"; tail -2 gpurun_out/drv_smoke.log
t0=$(date +%s); timeout 1800 python bench.py > gpurun_out/drv_bench.json 2> gpurun_out/drv_bench.err; echo "bench rc=$? $(( $(date +%s) - t0 ))s"
t0=$(date +%s); timeout 1800 python bench.py --impl reference > gpurun_out/drv_ref.json 2> gpurun_out/drv_ref.err; echo "ref rc=$? $(( $(date +%s) - t0 ))s"
python - <<'PY'
import json
for f in ("gpurun_out/drv_bench.json", "gpurun_out/drv_ref.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d.get("ms_per_step"), d.get("value"), (d.get("e2e") or {}).get("value"), d.get("steps"), d.get("warmup"),
          (d.get("cpu_baseline") or {}).get("value"), [ (r["preset"], r["threads"], round(r["seconds"],3)) for r in (d.get("reference_python") or {}).get("runs", [])])
PY
