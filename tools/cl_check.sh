#!/bin/bash
# d <= 32 tensor-core check: GPU tests, cfg5 lloyd (LK_TC2 = 1 / 0), hamerly, cfg1 forced TC.
O=gpurun_out/cl; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
for c in 1 0; do
  LK_TC2=$c python bench.py --workload cfg5 --strategy lloyd --steps 3 --warmup 3 --no-cpu > $O/c5_tc2_$c.json 2> $O/c5_tc2_$c.err; echo "tc2_$c=$?"
done
python bench.py --workload cfg5 --strategy hamerly --steps 3 --warmup 3 --no-cpu > $O/c5h.json 2> $O/c5h.err; echo "c5h=$?"
python bench.py --workload cfg1 --strategy lloyd --kernel tc --steps 3 --warmup 3 --no-cpu > $O/c1tc.json 2> $O/c1tc.err; echo "c1tc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assign_tc2 -s 2 -c 1 \
    -o $O/full_cfg5_tc2 python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 2 --no-cpu > $O/ncu.log 2>&1; echo "ncu=$?"
