#!/bin/bash
# quick iteration: tgy tests, cfg5 probe (phase clocks from iteration 6), A/B knobs
O=gpurun_out/${OUT:-r02i}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_tgy.py tests/test_gpu_fused.py -x -q > $O/pytest_tgy.log 2>&1; echo "tgy=$?"
LK_TGY_PROF=1 LK_TGY_PROF_SKIP=4 timeout 600 python tools/probe.py cfg5 ${T:-12} 0 yinyang:tc:0 > $O/cfg5_prof.jsonl 2> $O/cfg5_prof.err; echo "prof=$?"
timeout 600 python tools/probe.py cfg5 ${T:-12} 0 yinyang:tc:0 > $O/cfg5.jsonl 2> $O/cfg5.err; echo "probe=$?"
for v in $EXTRA; do
  env $v timeout 600 python tools/probe.py cfg5 ${T:-12} 0 yinyang:tc:0 > $O/cfg5_$v.jsonl 2> $O/cfg5_$v.err; echo "$v=$?"
done
