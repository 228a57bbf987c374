#!/bin/bash
# group-tile Yinyang: new tests, cfg5 probe
O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tgy.py -x -q > $O/pytest_tgy.log 2>&1; echo "tgy=$?"
timeout 900 python tools/probe.py cfg5 20 0 yinyang:tc:0 > $O/cfg5.jsonl 2> $O/cfg5.err; echo "cfg5=$?"
