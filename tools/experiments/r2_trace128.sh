#!/bin/bash
# score-kernel per-unit timeline at r_k 128 and 256 (clock64 marks)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for rk in 128 256; do
  PALU_SCORE_TRACE=1 timeout 300 python tools/score_trace.py --rank-k $rk --rank-v 256 > gpurun_out/score_trace_r$rk.txt 2>&1
done
