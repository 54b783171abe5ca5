ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_gaussblur.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launch_bench.log 2>&1; echo launches $?
ROUND=r01 bash tools/profile_all.sh
