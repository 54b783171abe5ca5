#!/bin/bash
# compute-sanitizer over the tiny-shape driver; summaries -> gpurun_out/sanitize_*.txt
python tools/sanitize_run.py > gpurun_out/sanitize_plain_run.txt 2>&1; echo plain $?; tail -1 gpurun_out/sanitize_plain_run.txt
for tool in memcheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo $tool $?; tail -3 gpurun_out/sanitize_$tool.txt
done
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 20 python tools/sanitize_run.py --quick > gpurun_out/sanitize_racecheck.txt 2>&1
echo racecheck $?; tail -3 gpurun_out/sanitize_racecheck.txt
PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 3 python tools/sanitize_run.py --canary > gpurun_out/sanitize_canary.txt 2>&1
echo canary $?; tail -3 gpurun_out/sanitize_canary.txt
