# r02i: GPU tests, bench C3 (+C2), reference arm C2
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_pytest.log 2>&1; tail -3 gpurun_out/r02i_pytest.log
timeout 900 python bench.py > gpurun_out/r02i_bench_c3.json 2> gpurun_out/r02i_bench_c3.err; echo bench_rc=$?
tail -c 2500 gpurun_out/r02i_bench_c3.json
timeout 600 python bench.py --config 2 > gpurun_out/r02i_bench_c2.json 2> gpurun_out/r02i_bench_c2.err; echo bench2_rc=$?
