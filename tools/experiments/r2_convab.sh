#!/bin/bash
# converter hand-off: release.cluster arrive (product) vs default-semantics arrive
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for a in "--bits 4" "--bits 2" "--rank-k 128 --rank-v 384 --bits 4"; do
  bash tools/ab_env.sh "X=1" "PALU_LIB_PATH=abtmp/convcta/libpalu_b200.so" --no-cpu --no-e2e --no-baseline $a
done 2>&1 | tee gpurun_out/r2_convab.txt
