#!/bin/bash
# Round-2 check: smoke, all GPU tests, default bench (+ reference arm), every workload,
# the self-launched 2-rank bench on one GPU, and the launch list of the default bench.
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench $?
cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo ref $?
STB200_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --workload jacobi3d --steps 5 --no-cpu-baseline > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err; echo share2 $?; tail -c 600 gpurun_out/bench_share2.json
bash tools/bench_all.sh gaussblur jacobi2d jacobi2d_paper gameoflife laplacian wave13pt jacobi3d divergence gradient tricubic uxx1 whispering lapgsrb tricubic2 > gpurun_out/bench_all.txt 2>&1; cat gpurun_out/bench_all.txt
