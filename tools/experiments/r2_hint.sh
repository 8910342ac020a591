#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for a in "" "--rank-k 128 --rank-v 384 --bits 16,4" "--bits 4" "--rope off"; do
  bash tools/ab_lib.sh abtmp/prev/libpalu_b200.so paper_2407_21118_b200/libpalu_b200.so $a
done 2>&1 | tee gpurun_out/r2_hint.txt
