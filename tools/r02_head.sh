#!/bin/bash
# HEAD check: smoke, GPU suite, default bench, cfg5 group-tile Yinyang full-size parity.
O=gpurun_out/${OUT:-r02h}; mkdir -p $O
git_head=${HEAD_HASH:-unknown}; echo $git_head > $O/head.txt
nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "bench=$?"
if [ -n "$PAR5" ]; then
  timeout 2400 python tools/fullsize_parity.py cfg5 --strategies ${PAR5} --rows 1000000 --all-rows-at none --out $O/fullsize_parity_cfg5.jsonl >> $O/parity5.log 2>&1; echo "par5=$?"
fi
