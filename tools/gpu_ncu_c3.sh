# full ncu captures of the two k_target launches on C3 (the bench config): seed and main
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"^k_target$" --launch-count 1 \
  -o gpurun_out/r02n_k_target_c3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02n_ncu_seed.log 2>&1; echo seed_rc=$?
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"^k_target$" --launch-skip 1 --launch-count 1 \
  -o gpurun_out/r02n_k_target_main_c3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02n_ncu_main.log 2>&1; echo main_rc=$?
for t in r02n_k_target_c3 r02n_k_target_main_c3; do ncu -i gpurun_out/$t.ncu-rep --page details > gpurun_out/${t}_details.txt 2>&1; done
python tools/traffic_json.py r02n 3
