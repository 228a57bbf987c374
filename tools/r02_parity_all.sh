#!/bin/bash
# Full-size parity of every quoted (config, strategy) at the commit in $LK_COMMIT
# (profiles/r02/fullsize_parity.jsonl): oracle re-decision per iteration, then the
# exhaustive tensor-core vs SIMT label comparisons.
O=gpurun_out/${OUT:-r02par}; mkdir -p $O
F=$O/fullsize_parity.jsonl
for spec in "cfg1:lloyd,yinyang:100000" "cfg2:lloyd,hamerly,yinyang:1000000" "cfg3:lloyd,hamerly,yinyang:250000" "cfg4:lloyd,hamerly,yinyang:250000"; do
  IFS=: read wl st rows <<< "$spec"
  timeout 2400 python tools/fullsize_parity.py $wl --strategies $st --rows $rows --out $F >> $O/parity.log 2>&1; echo "$wl=$?"
done
timeout 3000 python tools/fullsize_parity.py cfg5 --strategies lloyd,hamerly,yinyang --rows 1000000 --all-rows-at none --out $F >> $O/parity.log 2>&1; echo "cfg5=$?"
for spec in "cfg3:lloyd:30" "cfg4:lloyd:30" "cfg5:lloyd:20"; do
  IFS=: read wl st tm <<< "$spec"
  timeout 1800 python tools/fullsize_parity.py $wl --strategies $st --t-max $tm --tc-vs-simt --out $F >> $O/parity.log 2>&1; echo "simt_$wl=$?"
done
