# full ncu captures of the search launches on C3 (the bench config): k_target over the calibration sample,
# k_lane, k_target over what k_lane leaves
# usage: bash tools/gpu_ncu_c3.sh TAG
cd $GRAFT_REPO_ROOT
TAG=${1:-rXX}
mkdir -p gpurun_out
cap() {  # name regex skip
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"$2" --launch-skip $3 --launch-count 1 \
    -o gpurun_out/${TAG}_$1_c3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_ncu_$1.log 2>&1
  echo "$1 rc=$?"
  ncu -i gpurun_out/${TAG}_$1_c3.ncu-rep --page details > gpurun_out/${TAG}_$1_c3_details.txt 2>&1
}
cap k_target_sample "^k_target$" 0
cap k_lane "^k_lane$" 0
cap k_target_rest "^k_target$" 1
python tools/traffic_json.py $TAG 3
