timeout 1200 python -m pytest tests -x -q -m gpu -k "3d or dist or api" > gpurun_out/pytest_3d.log 2>&1; echo pytest $?; tail -2 gpurun_out/pytest_3d.log
bash tools/bench_all.sh laplacian wave13pt jacobi3d divergence gradient > gpurun_out/bench_3d.txt 2>&1; cat gpurun_out/bench_3d.txt
