#!/bin/bash
O=gpurun_out/${OUT:-r02san}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_fused.py -q -k simt_multikernel > $O/pytest_simt_mk.log 2>&1; echo "simt_mk=$?"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/sanitize_$tool.log 2>&1; echo "$tool=$?"
done
