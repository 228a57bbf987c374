#!/bin/bash
# ncu --set full of one launch of the kernels matching $K from a small-config bench run
O=gpurun_out/${OUT:-r02n}; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" --launch-skip ${SKIP:-8} --launch-count ${COUNT:-1} \
    -o $O/ncu_${TAG:-k} python bench.py --workload ${WL:-cfg1} --strategy yinyang --no-cpu > $O/ncu_${TAG:-k}.log 2>&1; echo "ncu=$?"
