#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
PALU_FUSED_TRACE=1 timeout 300 python tools/fused_trace.py --score-kernel tcgen05 > gpurun_out/vtrace_r256.txt 2>&1
PALU_FUSED_TRACE=1 timeout 300 python tools/fused_trace.py --score-kernel tcgen05 --rank-k 128 --rank-v 384 > gpurun_out/vtrace_preset.txt 2>&1
