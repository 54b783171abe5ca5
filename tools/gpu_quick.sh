# quick GPU check: full gpu tests + all-workload bench summary
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?; tail -2 gpurun_out/pytest_gpu.log
bash tools/bench_all.sh ${@} > gpurun_out/bench_all.txt 2>&1; cat gpurun_out/bench_all.txt
