#!/bin/bash
# TC-path check: GPU test suite, then lloyd/hamerly benches of the TC configs.
mkdir -p gpurun_out/tc
python -m pytest tests -m gpu -q -x > gpurun_out/tc/pytest_gpu.log 2>&1
echo "pytest=$?"
python bench.py --workload cfg5 --strategy lloyd --steps 3 --warmup 3 --no-cpu > gpurun_out/tc/b_cfg5_lloyd.json 2> gpurun_out/tc/b_cfg5_lloyd.err; echo "cfg5=$?"
python bench.py --workload cfg5 --strategy hamerly --steps 3 --warmup 3 --no-cpu > gpurun_out/tc/b_cfg5_hamerly.json 2> gpurun_out/tc/b_cfg5_hamerly.err; echo "cfg5h=$?"
python bench.py --workload cfg3 --strategy lloyd --steps 5 --warmup 3 --no-cpu > gpurun_out/tc/b_cfg3_lloyd.json 2> gpurun_out/tc/b_cfg3_lloyd.err; echo "cfg3=$?"
python bench.py --workload cfg4 --strategy lloyd --steps 5 --warmup 3 --no-cpu > gpurun_out/tc/b_cfg4_lloyd.json 2> gpurun_out/tc/b_cfg4_lloyd.err; echo "cfg4=$?"
if [ -n "$NCU5" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assign_tc -s 6 -c 1 \
    -o gpurun_out/tc/full_cfg5_tc python bench.py --workload cfg5 --strategy lloyd --steps 1 --warmup 3 --no-cpu \
    > gpurun_out/tc/ncu_full_cfg5.log 2>&1; echo "ncu=$?"
fi
