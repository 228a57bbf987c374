#!/bin/bash
O=gpurun_out/seed; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
python bench.py --no-cpu > $O/c2.json 2> $O/c2.err; echo "c2=$?"
python tools/e2e_phases.py cfg2 yinyang > $O/phases.txt 2>&1; echo "ph=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/e2e_phases.py cfg2 yinyang > /dev/null 2>&1; echo "l=$?"
