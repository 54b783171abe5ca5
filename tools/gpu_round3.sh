#!/bin/bash
# Round-2 (late) check: smoke, all GPU tests, default bench (auto variant) + reference arm,
# every workload, guard-band bounds checks.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench $?
cat gpurun_out/bench_default.json
bash tools/bench_all.sh gaussblur jacobi2d jacobi2d_paper jacobi2d9 jacobi2d_f64 gameoflife laplacian wave13pt jacobi3d divergence gradient tricubic uxx1 whispering lapgsrb tricubic2 > gpurun_out/bench_all.txt 2>&1; cat gpurun_out/bench_all.txt
bash tools/gpu_guard.sh
