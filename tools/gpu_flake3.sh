#!/bin/bash
STB200_LIB=expbuild/rel1/libstencil_b200.so timeout 1200 python tools/flake_hunt.py --kind jacobi2d5 --n 32768 --iters 10 --reps 10 --variants plain 2>&1 | tail -3
timeout 1200 python tools/flake_hunt.py --kind jacobi2d9 --n 32768 --iters 9 --reps 8 --variants plain,shuffle 2>&1 | tail -3
STB200_2D_NSW=3 timeout 1200 python tools/flake_hunt.py --kind gameoflife --n 16384 --iters 9 --reps 8 --dtype i32 --variants plain 2>&1 | tail -3
