#!/bin/bash
# A/B knobs: tensor-core pipeline (cfg5 lloyd) and the fused Yinyang path (cfg2).
O=gpurun_out/ab; mkdir -p $O
python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest=$?"
for v in "" "LK_TC_FAST=0" "LK_TC_SPIN=1" "LK_TC_ROT=1" "LK_TC_SPIN=1 LK_TC_ROT=1"; do
  tag=$(echo "base $v" | tr ' =' '__')
  env $v python bench.py --workload cfg5 --strategy lloyd --steps 2 --warmup 3 --no-cpu > $O/c5_$tag.json 2>/dev/null; echo "c5 $v $?"
done
for v in "" "LK_SGATE=0"; do
  tag=$(echo "base $v" | tr ' =' '__')
  env $v python bench.py --no-cpu > $O/c2_$tag.json 2>/dev/null; echo "c2 $v $?"
done
