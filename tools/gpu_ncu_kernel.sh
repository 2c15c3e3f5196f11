# one ncu --set full capture of a kernel in the C2 bench step: bash tools/gpu_ncu_kernel.sh TAG REGEX [SKIP] [CONFIG]
cd $GRAFT_REPO_ROOT
TAG=$1; RX=$2; SKIP=${3:-0}; CFG=${4:-2}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$RX --launch-skip $SKIP --launch-count 1 \
  -o gpurun_out/${TAG} python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}.log 2>&1
echo ncu_rc=$?
ncu -i gpurun_out/${TAG}.ncu-rep --page details > gpurun_out/${TAG}_details.txt 2>&1
