#!/bin/bash
# Second half of the round-end evidence (small outputs only): smoke, GPU tests,
# cfg3 / cfg4 benches, the cfg5 launch list and the k_assign_tc2 capture.
O=gpurun_out/prof2; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
python bench.py --workload cfg3 --strategy lloyd --steps 5 --warmup 3 --no-cpu > $O/b_cfg3_lloyd.json 2>/dev/null; echo "c3=$?"
python bench.py --workload cfg4 --strategy lloyd --steps 5 --warmup 3 --no-cpu > $O/b_cfg4_lloyd.json 2>/dev/null; echo "c4=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5.csv \
    python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 3 --no-cpu > $O/ncu_launches5.log 2>&1; echo "l5=$?"
timeout 900 ncu --set full --clock-control none -k regex:k_assign_tc2 -s 2 -c 1 \
    -o $O/full_cfg5_tc2 python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 2 --no-cpu \
    > $O/ncu_full_cfg5.log 2>&1; echo "n5=$?"
ls -la $O
