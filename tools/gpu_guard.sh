#!/bin/bash
# Bounds checks of our own (the pool refuses compute-sanitizer): guard-banded
# buffers + oracle parity over the tiny-shape suite, and the canary that must fire.
timeout 900 python tools/sanitize_run.py > gpurun_out/guard_run.txt 2>&1; echo guard $?; tail -2 gpurun_out/guard_run.txt
timeout 300 python tools/sanitize_run.py --canary > gpurun_out/guard_canary.txt 2>&1; echo canary $?; tail -2 gpurun_out/guard_canary.txt
