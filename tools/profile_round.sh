# Round profile capture on one GPU (run under gpurun): bench line, reference arm,
# ncu launch list, full-set captures of the two k_target launches (seeds, main).
# usage: bash tools/profile_round.sh TAG [CONFIG]
set -u
TAG=${1:-rXX}; CFG=${2:-2}
mkdir -p gpurun_out
python bench.py --config $CFG > gpurun_out/${TAG}_bench_c${CFG}.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
python bench.py --config $CFG --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_reference_c${CFG}.json 2> gpurun_out/${TAG}_ref.err; echo ref_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c${CFG}_launches.csv \
  python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_list.log 2>&1; echo list_rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_target -c 1 -o gpurun_out/${TAG}_k_target_c${CFG} \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_full.log 2>&1; echo full_rc=$?
ncu --set full --import-source on --clock-control none -k regex:k_target --launch-skip 1 --launch-count 1 \
  -o gpurun_out/${TAG}_k_target_main_c${CFG} \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_main.log 2>&1; echo main_rc=$?
