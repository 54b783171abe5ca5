#!/bin/bash
timeout 900 python -m pytest tests/test_coeffs_gpu.py -q -k "32768" -p no:cacheprovider 2>&1 | tail -3
timeout 900 python -m pytest tests/test_coeffs_gpu.py -q -k "32768" -p no:cacheprovider 2>&1 | tail -3
timeout 900 python tools/flake_hunt.py --kind jacobi2d5 --n 32768 --iters 10 --reps 8 2>&1 | tail -6
timeout 900 python tools/flake_hunt.py --kind gaussblur5x5 --n 8192 --iters 100 --reps 12 2>&1 | tail -4
timeout 900 python tools/flake_hunt.py --kind gameoflife --n 16384 --iters 10 --reps 12 --dtype i32 2>&1 | tail -4
