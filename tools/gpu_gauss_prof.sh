for v in shuffle plain; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k2d2 -s 1 -c 1 -f -o gpurun_out/prof_gauss_pair_$v python tools/prof_run.py --workload gaussblur --variant $v --run --fusion 2 > /dev/null 2>&1; echo $v $?
done
