#!/bin/bash
# GPU suite + cfg5 full-size parity
O=gpurun_out/${OUT:-r02k}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
if [ -n "$PAR5" ]; then
  timeout 2400 python tools/fullsize_parity.py cfg5 --strategies ${PAR5} --rows 1000000 --all-rows-at none --out $O/fullsize_parity_cfg5.jsonl >> $O/parity5.log 2>&1; echo "par5=$?"
fi
