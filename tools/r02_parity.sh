#!/bin/bash
# full-size parity at HEAD (profiles/r02/fullsize_parity.jsonl)
O=gpurun_out/${OUT:-r02par}; mkdir -p $O
F=$O/fullsize_parity.jsonl
for spec in ${SPECS:-"cfg1:lloyd,yinyang:100000" "cfg2:lloyd,hamerly,yinyang:1000000" "cfg3:lloyd,hamerly,yinyang:250000" "cfg4:lloyd,hamerly,yinyang:250000"}; do
  IFS=: read wl st rows <<< "$spec"
  timeout 2400 python tools/fullsize_parity.py $wl --strategies $st --rows $rows --out $F >> $O/parity.log 2>&1; echo "$wl=$?"
done
for spec in ${SIMT:-}; do
  IFS=: read wl st tm <<< "$spec"
  timeout 1800 python tools/fullsize_parity.py $wl --strategies $st --t-max $tm --tc-vs-simt --out $F >> $O/parity.log 2>&1; echo "simt_$wl=$?"
done
