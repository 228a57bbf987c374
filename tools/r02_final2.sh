#!/bin/bash
# Final check at the round's last commit: GPU suite, smoke, default bench + reference arm,
# cfg5 group-tile Yinyang full-size parity.
O=gpurun_out/${OUT:-r02z}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > $O/bench_cfg5_yinyang.json 2> $O/bench_cfg5.err; echo "bench=$?"
timeout 600 python bench.py --impl reference > $O/bench_reference_cfg5.json 2> $O/bench_ref.err; echo "ref=$?"
timeout 2400 python tools/fullsize_parity.py cfg5 --strategies yinyang --rows 1000000 --all-rows-at none --out $O/fullsize_parity_cfg5.jsonl >> $O/parity5.log 2>&1; echo "par5=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_yy_fused" --launch-skip 4 --launch-count 1 \
    -o $O/ncu_full_cfg2_fused python bench.py --workload cfg2 --strategy yinyang --steps 2 --warmup 3 --no-cpu > $O/ncu_full_2.log 2>&1; echo "ncu_2=$?"
