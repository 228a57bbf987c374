#!/bin/bash
# Elkan (per-centroid bounds) and Regroup as distinct variants: bench lines and full-size parity
O=gpurun_out/${OUT:-r02v}; mkdir -p $O
for spec in cfg1:elkan cfg1:regroup cfg2:regroup cfg2:hamerly cfg1:hamerly; do
  IFS=: read wl st <<< "$spec"
  timeout 600 python bench.py --workload $wl --strategy $st --no-cpu > $O/b_${wl}_${st}.json 2> $O/b_${wl}_${st}.err; echo "b_$spec=$?"
done
timeout 1200 python tools/fullsize_parity.py cfg1 --strategies hamerly,elkan,regroup --rows 100000 --out $O/fullsize_parity_variants.jsonl >> $O/parity.log 2>&1; echo "p1=$?"
timeout 1800 python tools/fullsize_parity.py cfg2 --strategies regroup --rows 1000000 --out $O/fullsize_parity_variants.jsonl >> $O/parity.log 2>&1; echo "p2=$?"
