H="timeout 1200 python tools/flake_hunt.py"
$H --kind jacobi2d5 --n 32768 --iters 10 --reps 8 2>&1 | tail -1
$H --kind jacobi2d9 --n 32768 --iters 9 --reps 6 2>&1 | tail -1
$H --kind gaussblur5x5 --n 8192 --iters 100 --reps 10 2>&1 | tail -1
$H --kind gameoflife --n 16384 --iters 10 --reps 8 --dtype i32 2>&1 | tail -1
bash tools/bench_all.sh gaussblur jacobi2d_paper gameoflife
