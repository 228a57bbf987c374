#!/bin/bash
# one ncu --set full capture of the kernels matching $K (regex) from the cfg5 probe
O=gpurun_out/${OUT:-r02n}; mkdir -p $O
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$K" --launch-skip ${SKIP:-6} --launch-count ${COUNT:-1} \
    -o $O/ncu_${TAG:-k} python tools/probe.py cfg5 ${T:-9} 0 yinyang:tc:0 > $O/ncu_${TAG:-k}.log 2>&1; echo "ncu=$?"
