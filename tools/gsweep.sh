# sweep + GPU tests, printing the test summary last (usage: bash tools/gsweep.sh SETTING...)
bash tools/sweep.sh "$@" > gpurun_out/s.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.txt 2>&1
cat gpurun_out/s.txt; tail -1 gpurun_out/t.txt
