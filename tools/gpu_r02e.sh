cd $GRAFT_REPO_ROOT
export SPH_GROUP_G=${G:-4}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_c2_launches.csv \
  python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02e_ncu_list.log 2>&1; echo list_rc=$?
python tools/launches.py gpurun_out/r02e_c2_launches.csv 36 2>&1 | grep -v "^ *[0-9.]* us  x1 \| k_ffma" | tail -40
bash tools/gpu_ncu_kernel.sh r02e_k_group k_group 0 2
