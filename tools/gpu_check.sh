#!/bin/bash
# full GPU test suite + smoke + sanitizer canary; args: extra commands are not taken
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?; tail -3 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?; tail -5 gpurun_out/pytest_gpu.log
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python tools/sanitize_run.py --canary > gpurun_out/sanitize_canary.txt 2>&1
echo canary $?; grep -c "Invalid" gpurun_out/sanitize_canary.txt; tail -2 gpurun_out/sanitize_canary.txt
