mkdir -p gpurun_out/p1
timeout 900 python tools/probe.py cfg5 20 0 lloyd:tc:0 hamerly:tc:0 yinyang:simt:32 yinyang:simt:16 yinyang:tc:32 > gpurun_out/p1/cfg5.jsonl 2> gpurun_out/p1/cfg5.err; echo "cfg5=$?"
timeout 600 python tools/probe.py cfg3 30 0 lloyd:tc:0 yinyang:tc:0 hamerly:tc:0 yinyang:simt:32 > gpurun_out/p1/cfg3.jsonl 2> gpurun_out/p1/cfg3.err; echo "cfg3=$?"
nproc > gpurun_out/p1/nproc.txt; free -g >> gpurun_out/p1/nproc.txt; lscpu >> gpurun_out/p1/nproc.txt
