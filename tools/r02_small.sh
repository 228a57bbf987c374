#!/bin/bash
# cfg1 / cfg2 bench lines (fused SIMT Yinyang) + the fused-path tests
O=gpurun_out/${OUT:-r02sm}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_fused.py -x -q > $O/pytest_fused.log 2>&1; echo "fused=$?"
for wl in cfg2 cfg1; do
  for rep in 1 2; do
    timeout 600 python bench.py --workload $wl --strategy yinyang --no-cpu > $O/b_${wl}_$rep.json 2> $O/b_${wl}_$rep.err; echo "$wl=$?"
  done
done
