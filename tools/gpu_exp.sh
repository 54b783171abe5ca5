timeout 1200 python -m pytest tests -x -q -m gpu -k "3d or dist" > gpurun_out/pytest_3d.log 2>&1; echo pytest $?; tail -2 gpurun_out/pytest_3d.log
for b in 1 0; do echo "STG=$b"; STB200_STG=$b bash tools/bench_all.sh laplacian wave13pt jacobi3d gradient; done
