#!/bin/bash
# timing probes of the group-tile pass: iteration 8's pass (launch 7) with one part switched off
O=gpurun_out/${OUT:-r02d}; mkdir -p $O
for v in 0 1 2 3 4; do
  LK_TGY_DBG=$v LK_TGY_DBG_AT=7 timeout 300 python tools/probe.py cfg5 8 0 yinyang:tc:0 > $O/dbg$v.jsonl 2> $O/dbg$v.err; echo "dbg$v=$?"
done
