#!/bin/bash
# PDL check: GPU tests, cfg2 / cfg1 benches with LK_PDL = 1 / 0.
O=gpurun_out/pdl; mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest=$?"
for v in 1 0 1; do
  LK_PDL=$v python bench.py --no-cpu > $O/c2_pdl$v.json 2> $O/c2_pdl$v.err; echo "c2 pdl$v=$?"
done
for v in 1 0; do
  LK_PDL=$v python bench.py --workload cfg1 --no-cpu > $O/c1_pdl$v.json 2> $O/c1_pdl$v.err; echo "c1 pdl$v=$?"
done
