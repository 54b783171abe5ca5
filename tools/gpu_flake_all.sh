#!/bin/bash
# race hunt over every streaming / staged kernel family (default build)
H="timeout 1200 python tools/flake_hunt.py"
$H --kind jacobi2d5 --n 32768 --iters 10 --reps 8 2>&1 | tail -1
$H --kind jacobi2d9 --n 32768 --iters 9 --reps 8 2>&1 | tail -1
$H --kind gaussblur5x5 --n 8192 --iters 100 --reps 10 2>&1 | tail -1
$H --kind gameoflife --n 16384 --iters 10 --reps 8 --dtype i32 2>&1 | tail -1
$H --kind laplacian3d7 --shape 256,256,512 --iters 10 --reps 8 --dtype f64 2>&1 | tail -1
$H --kind wave13pt --shape 256,256,512 --iters 10 --reps 8 --dtype f64 2>&1 | tail -1
$H --kind divergence --shape 256,256,512 --iters 4 --reps 8 2>&1 | tail -1
$H --kind tricubic --shape 256,256,256 --iters 4 --reps 8 2>&1 | tail -1
$H --kind lapgsrb --shape 256,512,512 --iters 6 --reps 8 2>&1 | tail -1
