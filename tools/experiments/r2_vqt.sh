#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
PALU_FUSED_TRACE=1 timeout 300 python tools/vq_trace.py --rank-k 256 --rank-v 256 --bits 4 --ctas 0,73 > gpurun_out/vqt_int4.txt 2>&1
PALU_FUSED_TRACE=1 timeout 300 python tools/vq_trace.py --rank-k 128 --rank-v 384 --bits 16,4 --ctas 0,73 > gpurun_out/vqt_k16v4.txt 2>&1
