#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for rk in 128 256; do
  PALU_LIB_PATH=abtmp/diag/libpalu_b200.so PALU_SCORE_TRACE=1 timeout 300 python tools/score_trace.py --rank-k $rk --rank-v 256 > gpurun_out/score_trace_e5_r$rk.txt 2>&1
done
for m in 1 4 5; do
  echo "== mode $m"; PALU_LIB_PATH=abtmp/diag/libpalu_b200.so PALU_TC_PROFILE_MODE=$m PALU_SCORE_TRACE=1 timeout 120 python tools/score_trace.py --rank-k 128 --rank-v 256 2>&1 | grep -E "rope_score|MMA loop|issue span us|wake|idle|exchange"
done > gpurun_out/score_modes_e5.txt 2>&1
