#!/bin/bash
# k_assign_tgy phase clocks (LK_TGY_PROF) over a cfg5 Yinyang trajectory + per-iteration probe
O=gpurun_out/${OUT:-r02p}; mkdir -p $O
timeout 600 python tools/probe.py cfg5 ${T:-12} 0 yinyang:tc:0 > $O/cfg5.jsonl 2> $O/cfg5.err; echo "probe=$?"
LK_TGY_PROF=1 timeout 600 python tools/probe.py cfg5 ${T:-12} 0 yinyang:tc:0 > $O/cfg5_prof.jsonl 2> $O/cfg5_prof.err; echo "prof=$?"
for v in $EXTRA; do
  env $v timeout 600 python tools/probe.py cfg5 ${T:-12} 0 yinyang:tc:0 > $O/cfg5_$v.jsonl 2> $O/cfg5_$v.err; echo "$v=$?"
done
