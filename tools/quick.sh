#!/bin/bash
# quick GPU check: smoke, GPU tests, cfg5 / cfg3 / cfg4 lloyd benches, cfg5 launch list
O=gpurun_out/q; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
for c in cfg5 cfg3 cfg4; do
  python bench.py --workload $c --strategy lloyd --steps 3 --warmup 3 --no-cpu > $O/b_${c}_lloyd.json 2> $O/b_$c.err; echo "$c=$?"
done
python bench.py --workload cfg5 --strategy hamerly --steps 3 --warmup 3 --no-cpu > $O/b_cfg5_hamerly.json 2>/dev/null; echo "c5h=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
    python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 3 --no-cpu > $O/ncu_launches5.log 2>&1; echo "l5=$?"
