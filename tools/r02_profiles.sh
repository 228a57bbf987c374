#!/bin/bash
# Round-2 evidence: GPU suite, smoke, default bench + reference arm, other configs,
# ncu launch list and --set full captures (cfg5 Yinyang, cfg5 Hamerly filter, cfg2 fused path).
O=gpurun_out/${OUT:-r02prof}; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
  python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
fi
timeout 900 python bench.py > $O/bench_cfg5_yinyang.json 2> $O/bench_cfg5.err; echo "bench=$?"
timeout 600 python bench.py --impl reference > $O/bench_reference_cfg5.json 2> $O/bench_ref.err; echo "ref=$?"
for spec in cfg1:yinyang cfg2:yinyang cfg3:lloyd cfg3:yinyang cfg4:lloyd cfg4:yinyang cfg5:lloyd cfg5:hamerly; do
  IFS=: read wl st <<< "$spec"
  timeout 600 python bench.py --workload $wl --strategy $st --no-cpu > $O/b_${wl}_${st}.json 2> $O/b_${wl}_${st}.err; echo "b_$spec=$?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launches.log 2>&1; echo "launches=$?"
timeout 1500 ncu --set full --clock-control none \
    -k regex:"k_assign_tgy|k_filter_tgy|k_sort_gather|k_assign_tc|k_recheck_cand|k_sort_hist" --launch-skip 18 --launch-count 6 \
    -o $O/ncu_full_cfg5 python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu_full=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_filter_hamerly_tc" --launch-skip 3 --launch-count 1 \
    -o $O/ncu_full_cfg5_hamerly python bench.py --workload cfg5 --strategy hamerly --steps 2 --warmup 3 --no-cpu > $O/ncu_full_h.log 2>&1; echo "ncu_h=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_yy_fused|k_update_centroids|k_half_sep" --launch-skip 12 --launch-count 3 \
    -o $O/ncu_full_cfg2 python bench.py --workload cfg2 --strategy yinyang --steps 2 --warmup 3 --no-cpu > $O/ncu_full_2.log 2>&1; echo "ncu_2=$?"
ls -la $O/*.ncu-rep
