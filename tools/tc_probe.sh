#!/bin/bash
# Timing probes of the centered d = 32 tensor-core pass (iteration 2; labels are
# wrong under a probe).  LK_TC_DBG=1: no epilogue work; 2: no MMAs; 3: neither.
O=gpurun_out/probe; mkdir -p $O
for v in "0 1" "3 1" "3 2" "3 4" "1 1" "1 2" "0 2"; do
  set -- $v
  LK_TC_DBG=$1 LK_TC_CL=$2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_assign_tc -s 2 -c 1 --csv \
    python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 1 --no-cpu > $O/ncu_dbg$1_cl$2.csv 2>$O/ncu_dbg$1_cl$2.err; echo "dbg$1 cl$2 $?"
done
