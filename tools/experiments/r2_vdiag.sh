#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for m in 0 1 3; do
  echo "== PALU_VALUE_DIAG=$m"
  PALU_LIB_PATH=abtmp/diag/libpalu_b200.so PALU_VALUE_DIAG=$m PALU_FUSED_TRACE=1 timeout 300 python tools/fused_trace.py --score-kernel tcgen05 2>&1 | grep -E "palu_value|^value|landed|end by" | cut -c1-300
done > gpurun_out/vdiag.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"value_tc_kernel|value_merge|rope_score" -c 6 python tools/fused_trace.py --score-kernel tcgen05 2>&1 | grep -E "value_tc_kernel|value_merge|rope_score|gpu__time_duration|dram__bytes" | head -24 >> gpurun_out/vdiag.txt
