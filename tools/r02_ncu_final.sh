#!/bin/bash
# ncu --set full summaries at the round's last commit (profiles/r02/ncu_full_summary.json)
O=gpurun_out/${OUT:-r02ncu}; mkdir -p $O
timeout 1500 ncu --set full --clock-control none \
    -k regex:"k_assign_tgy|k_filter_tgy|k_sort_gather|k_assign_tc|k_recheck_cand|k_sort_hist" --launch-skip 18 --launch-count 6 \
    -o $O/ncu_full_cfg5 python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_full.log 2>&1; echo "ncu_full=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_filter_hamerly_tc" --launch-skip 3 --launch-count 1 \
    -o $O/ncu_full_cfg5_hamerly python bench.py --workload cfg5 --strategy hamerly --steps 2 --warmup 3 --no-cpu > $O/ncu_full_h.log 2>&1; echo "ncu_h=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_assign_tc2" --launch-skip 0 --launch-count 1 \
    -o $O/ncu_full_cfg5_tc2 python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 3 --no-cpu > $O/ncu_full_tc2.log 2>&1; echo "ncu_tc2=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_yy_fused|k_update_centroids|k_half_sep" --launch-skip 12 --launch-count 3 \
    -o $O/ncu_full_cfg2 python bench.py --workload cfg2 --strategy yinyang --steps 2 --warmup 3 --no-cpu > $O/ncu_full_2.log 2>&1; echo "ncu_2=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_half_sep|k_update_centroids" --launch-skip 6 --launch-count 2 \
    -o $O/ncu_full_cfg4 python bench.py --workload cfg4 --strategy yinyang --steps 2 --warmup 3 --no-cpu > $O/ncu_full_4.log 2>&1; echo "ncu_4=$?"
ls -la $O/*.ncu-rep
