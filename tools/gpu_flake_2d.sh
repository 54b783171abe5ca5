#!/bin/bash
# race hunt over the streaming 2-D kernels (both variants, default build)
H="timeout 1200 python tools/flake_hunt.py"
$H --kind jacobi2d5 --n 32768 --iters 10 --reps 8 2>&1 | tail -1
$H --kind jacobi2d9 --n 32768 --iters 10 --reps 8 2>&1 | tail -1
$H --kind gaussblur5x5 --n 8192 --iters 100 --reps 10 2>&1 | tail -1
$H --kind jacobi2d5 --n 16384 --iters 9 --reps 6 --dtype f64 2>&1 | tail -1
$H --kind gameoflife --n 16384 --iters 10 --reps 6 --dtype i32 2>&1 | tail -1
