#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "norope" 2>&1 | tail -1
PALU_PARITY_LOG=gpurun_out/r02_parity_lsq.jsonl timeout 600 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -x -k "norope_r256_int4" 2>&1 | tail -1
PALU_LIB_PATH=abtmp/diag/libpalu_b200.so timeout 300 python tools/lsq_trace.py > gpurun_out/lsq_trace4.txt 2>&1
for rep in 1 2; do
for lib in abtmp/prev paper_2407_21118_b200; do
  for b in 4 8; do
  v=$(PALU_LIB_PATH=$lib/libpalu_b200.so timeout 150 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-baseline --rope off --bits $b 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['per_kernel_ms']['palu_latent_score_tc']*1e3,1))")
  echo "$lib bits $b: $v"
  done
done; done 2>&1 | tee gpurun_out/r2_lsq5.txt
