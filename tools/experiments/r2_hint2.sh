#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
for a in "" "--rank-k 128 --rank-v 384 --bits 16,4" "--bits 4" "--rope off --bits 4" "--rank-k 128 --rank-v 384"; do
  bash tools/ab_lib.sh abtmp/prev/libpalu_b200.so paper_2407_21118_b200/libpalu_b200.so $a
done 2>&1 | tee gpurun_out/r2_hint3.txt
