#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for i in 1 2 3 4; do
  timeout 500 python -m pytest tests/test_gpu_parity.py -q -m gpu -rf -p no:cacheprovider 2>&1 | grep -E "FAILED|passed|failed|assert|Error" | head -12
done 2>&1 | tee gpurun_out/flaky.txt
