#!/bin/bash
# group-tile Yinyang: new tests, cfg5 probe, ncu of the tgy pass
O=gpurun_out/${OUT:-r02f}; mkdir -p $O
timeout 420 python -m pytest tests/test_gpu_tgy.py -x -q > $O/pytest_tgy.log 2>&1; echo "tgy=$?"
timeout 420 python tools/probe.py cfg5 20 0 yinyang:tc:0 > $O/cfg5.jsonl 2> $O/cfg5.err; echo "cfg5=$?"
if [ -n "$NCU" ]; then
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_assign_tgy|k_filter_tgy|k_sort_gather|k_tile_labels" --launch-skip 32 --launch-count 4 -o $O/tgy python tools/probe.py cfg5 12 0 yinyang:tc:0 > $O/ncu.log 2>&1; echo "ncu=$?"
fi
