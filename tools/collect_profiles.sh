#!/bin/bash
# Round-end evidence: bench lines (ours + reference arm), per-config benches,
# the ncu launch list of the default bench, and `ncu --set full` captures of
# the dominant kernels.  Everything lands in gpurun_out/prof/.
#   gpurun -- 'bash tools/collect_profiles.sh'
set -u
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
python bench.py --impl reference > $O/bench_reference_cfg2.json 2> $O/bench_reference_cfg2.err
python bench.py --workload cfg1 --no-cpu > $O/b_cfg1_yinyang.json 2>/dev/null
python bench.py --workload cfg3 --strategy lloyd --steps 5 --warmup 3 --no-cpu > $O/b_cfg3_lloyd.json 2>/dev/null
python bench.py --workload cfg3 --strategy yinyang --steps 5 --warmup 3 --no-cpu > $O/b_cfg3_yinyang.json 2>/dev/null
python bench.py --workload cfg4 --strategy lloyd --steps 5 --warmup 3 --no-cpu > $O/b_cfg4_lloyd.json 2>/dev/null
python bench.py --workload cfg5 --strategy lloyd --steps 3 --warmup 3 --no-cpu > $O/b_cfg5_lloyd.json 2>/dev/null
python bench.py --workload cfg5 --strategy hamerly --steps 3 --warmup 3 --no-cpu > $O/b_cfg5_hamerly.json 2>/dev/null
# launch list of the default bench (cold-cache, serialised per-launch durations)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_launches.log 2>&1
# full captures of the dominant kernels
ncu --set full --clock-control none --import-source on -k regex:k_yy_fused -s 12 -c 1 \
    -o $O/full_cfg2_fused python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_full_cfg2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_assign_tc -s 4 -c 1 \
    -o $O/full_cfg3_tc python bench.py --workload cfg3 --strategy lloyd --steps 1 --warmup 3 --no-cpu \
    > $O/ncu_full_cfg3.log 2>&1
echo collected
