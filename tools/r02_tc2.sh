#!/bin/bash
# k_assign_tc2 change: parity tests on the tensor-core paths, cfg5 Lloyd / Hamerly / Yinyang lines
O=gpurun_out/${OUT:-r02tc2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tgy.py tests/test_gpu_fused.py -q -x > $O/pytest.log 2>&1; echo "t=$?"
for st in lloyd hamerly; do
  timeout 600 python bench.py --workload cfg5 --strategy $st --no-cpu > $O/b_cfg5_$st.json 2> $O/b_cfg5_$st.err; echo "b_$st=$?"
done
timeout 600 python tools/probe.py cfg5 8 0 yinyang:tc:0 > $O/cfg5_yy.jsonl 2> $O/cfg5_yy.err; echo "probe=$?"
