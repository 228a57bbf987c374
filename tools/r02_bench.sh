#!/bin/bash
O=gpurun_out/${OUT:-r02bench}; mkdir -p $O
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref=$?"
