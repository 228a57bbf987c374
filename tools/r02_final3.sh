#!/bin/bash
# Final evidence at the round's last commit ($LK_COMMIT): GPU suite, smoke, default bench +
# reference arm, cfg5 Lloyd / Hamerly lines, launch list, cfg5 full-size parity (all three
# strategies + tensor-core vs SIMT).
O=gpurun_out/${OUT:-r02zz}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > $O/bench_cfg5_yinyang.json 2> $O/bench_cfg5.err; echo "bench=$?"
timeout 600 python bench.py --impl reference > $O/bench_reference_cfg5.json 2> $O/bench_ref.err; echo "ref=$?"
for st in lloyd hamerly; do
  timeout 600 python bench.py --workload cfg5 --strategy $st --no-cpu > $O/b_cfg5_$st.json 2> $O/b_cfg5_$st.err; echo "b_$st=$?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launches.log 2>&1; echo "launches=$?"
timeout 900 ncu --set full --clock-control none -k regex:"k_assign_tc2" --launch-skip 0 --launch-count 1 \
    -o $O/ncu_full_cfg5_tc2 python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 3 --no-cpu > $O/ncu_full_tc2.log 2>&1; echo "ncu_tc2=$?"
timeout 3000 python tools/fullsize_parity.py cfg5 --strategies lloyd,hamerly,yinyang --rows 1000000 --all-rows-at none --out $O/fullsize_parity_cfg5.jsonl >> $O/parity5.log 2>&1; echo "par5=$?"
timeout 1800 python tools/fullsize_parity.py cfg5 --strategies lloyd --t-max 20 --tc-vs-simt --out $O/fullsize_parity_cfg5.jsonl >> $O/parity5.log 2>&1; echo "simt5=$?"
