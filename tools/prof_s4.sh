#!/bin/bash
# Session-4 profiling payload: launch list of cfg2 and cfg5 (lloyd), and
# `ncu --set full` captures (with source) of the fused Yinyang kernel (cfg2)
# and the d = 32 tensor-core assignment (cfg5).  Outputs in gpurun_out/p4/.
set -u
O=gpurun_out/p4
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_launches_cfg2.log 2>&1
echo launches2=$?
ncu --set full --clock-control none --import-source on -k regex:k_yy_fused -s 12 -c 1 \
    -o $O/full_cfg2_fused python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_full_cfg2.log 2>&1
echo full2=$?
ncu --set full --clock-control none --import-source on -k regex:"k_update|k_half_sep|k_recheck_fp64" -s 30 -c 3 \
    -o $O/full_cfg2_small python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_small_cfg2.log 2>&1
echo small2=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
    python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 3 --no-cpu > $O/ncu_launches_cfg5.log 2>&1
echo launches5=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_assign_tc -s 6 -c 2 \
    -o $O/full_cfg5_tc python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 3 --no-cpu \
    > $O/ncu_full_cfg5.log 2>&1
echo full5=$?
