#!/bin/bash
# One gpurun payload: smoke, GPU test suite, default bench, and short benches
# of the configs given as arguments.  Outputs land in gpurun_out/.
#   gpurun -- 'bash tools/gpu_check.sh cfg1 cfg5'
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke=$?"
if [ -z "$SKIP_TESTS" ]; then
  python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest=$?"
fi
python bench.py ${BENCH_ARGS:---no-cpu} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench=$?"
for c in "$@"; do
  python bench.py --workload "$c" --steps 3 --warmup 3 --no-cpu > "gpurun_out/b_$c.json" 2> "gpurun_out/b_$c.err"
  echo "bench_$c=$?"
done
