#!/bin/bash
# Round-end evidence: smoke, GPU tests, bench lines (ours + reference arm),
# per-config benches, ncu launch lists (cfg2, cfg5) and `ncu --set full`
# captures of the dominant kernels.  Everything lands in gpurun_out/final/
# (kept under gpurun's 64 MiB merge limit: only the cfg2 capture carries source).
#   gpurun -- 'bash tools/collect_profiles.sh'
set -u
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench=$?"
python bench.py --impl reference > $O/bench_reference_cfg2.json 2> $O/bench_reference_cfg2.err; echo "ref=$?"
python bench.py --workload cfg1 --no-cpu > $O/b_cfg1_yinyang.json 2>/dev/null
python bench.py --workload cfg3 --strategy lloyd --steps 5 --warmup 3 --no-cpu > $O/b_cfg3_lloyd.json 2>/dev/null
python bench.py --workload cfg3 --strategy yinyang --steps 5 --warmup 3 --no-cpu > $O/b_cfg3_yinyang.json 2>/dev/null
python bench.py --workload cfg4 --strategy lloyd --steps 5 --warmup 3 --no-cpu > $O/b_cfg4_lloyd.json 2>/dev/null
python bench.py --workload cfg5 --strategy lloyd --steps 3 --warmup 3 --no-cpu > $O/b_cfg5_lloyd.json 2>/dev/null
python bench.py --workload cfg5 --strategy hamerly --steps 3 --warmup 3 --no-cpu > $O/b_cfg5_hamerly.json 2>/dev/null
echo "benches done"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_launches2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
    python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 3 --no-cpu > $O/ncu_launches5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_yy_fused -s 12 -c 1 \
    -o $O/full_cfg2_fused python bench.py --steps 3 --warmup 3 --no-cpu > $O/ncu_full_cfg2.log 2>&1
ncu --set full --clock-control none -k regex:k_assign_tc -s 4 -c 1 \
    -o $O/full_cfg3_tc python bench.py --workload cfg3 --strategy lloyd --steps 1 --warmup 3 --no-cpu \
    > $O/ncu_full_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_assign_tc2|k_filter_hamerly_tc" -s 2 -c 2 \
    -o $O/full_cfg5 python bench.py --workload cfg5 --strategy hamerly --steps 1 --warmup 2 --no-cpu \
    > $O/ncu_full_cfg5.log 2>&1
echo collected
ls -la $O | tail -30
