#!/bin/bash
# Everything at the round's last commit ($LK_COMMIT): GPU suite, smoke, every bench line,
# the launch list, full-size parity of every quoted (config, strategy) + TC vs SIMT + variants.
O=gpurun_out/${OUT:-r02end}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > $O/bench_cfg5_yinyang.json 2> $O/bench_cfg5.err; echo "bench=$?"
timeout 600 python bench.py --impl reference > $O/bench_reference_cfg5.json 2> $O/bench_ref.err; echo "ref=$?"
for spec in cfg1:yinyang cfg1:hamerly cfg1:elkan cfg1:regroup cfg2:yinyang cfg2:hamerly cfg2:regroup cfg3:lloyd cfg3:yinyang cfg4:lloyd cfg4:yinyang cfg5:lloyd cfg5:hamerly; do
  IFS=: read wl st <<< "$spec"
  timeout 600 python bench.py --workload $wl --strategy $st --no-cpu > $O/b_${wl}_${st}.json 2> $O/b_${wl}_${st}.err; echo "b_$spec=$?"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launches.log 2>&1; echo "launches=$?"
OUT=${OUT:-r02end} bash tools/r02_parity_all.sh
timeout 1200 python tools/fullsize_parity.py cfg1 --strategies hamerly,elkan,regroup --rows 100000 --out $O/fullsize_parity.jsonl >> $O/parity.log 2>&1; echo "v1=$?"
timeout 1800 python tools/fullsize_parity.py cfg2 --strategies regroup --rows 1000000 --out $O/fullsize_parity.jsonl >> $O/parity.log 2>&1; echo "v2=$?"
