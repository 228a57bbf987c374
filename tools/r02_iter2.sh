#!/bin/bash
# tgy/fused tests, cfg5 probe per filter variant
O=gpurun_out/${OUT:-r02k}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_tgy.py tests/test_gpu_fused.py -x -q > $O/pytest_tgy.log 2>&1; echo "tgy=$?"
timeout 600 python tools/probe.py cfg5 ${T:-12} 0 yinyang:tc:0 > $O/cfg5.jsonl 2> $O/cfg5.err; echo "probe=$?"
for v in $EXTRA; do
  env $v timeout 600 python tools/probe.py cfg5 ${T:-12} 0 yinyang:tc:0 > $O/cfg5_$v.jsonl 2> $O/cfg5_$v.err; echo "$v=$?"
done
if [ -n "$SUITE" ]; then timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "suite=$?"; fi
