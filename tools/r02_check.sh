#!/bin/bash
# Round-2 GPU check: smoke, GPU suite, cfg5/cfg3 per-iteration probes.
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1; nproc > $O/nproc.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 900 python tools/probe.py cfg5 20 0 lloyd:tc:0 hamerly:tc:0 yinyang:simt:32 yinyang:simt:16 > $O/cfg5.jsonl 2> $O/cfg5.err; echo "cfg5=$?"
timeout 600 python tools/probe.py cfg3 30 0 lloyd:tc:0 yinyang:tc:0 hamerly:tc:0 > $O/cfg3.jsonl 2> $O/cfg3.err; echo "cfg3=$?"
timeout 300 python bench.py --no-cpu > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench=$?"
