#!/bin/bash
# half-separation tile sizes: the bounded-strategy tests + cfg4 / cfg1 / cfg2 / cfg3 lines
O=gpurun_out/${OUT:-r02hs}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
for spec in cfg4:yinyang cfg4:hamerly cfg1:yinyang cfg1:hamerly cfg2:yinyang cfg3:yinyang; do
  IFS=: read wl st <<< "$spec"
  timeout 600 python bench.py --workload $wl --strategy $st --no-cpu > $O/b_${wl}_${st}.json 2> $O/b_${wl}_${st}.err; echo "b_$spec=$?"
done
