#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
PALU_PARITY_LOG=gpurun_out/r02_parity_merge.jsonl timeout 600 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -x -k "r256_bf16_64k or preset_k16v4 or gqa8_r64_bf16" 2>&1 | tail -1
for a in "" "--rank-k 128 --rank-v 384 --bits 16,4"; do
  bash tools/ab_lib.sh abtmp/prev/libpalu_b200.so paper_2407_21118_b200/libpalu_b200.so $a
done 2>&1 | tee gpurun_out/r2_merge.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:value_merge -c 4 python bench.py --steps 1 --warmup 2 --no-cpu --no-e2e --no-baseline --layers 2 2>&1 | grep -E "gpu__time" | head -4
