#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "norope" 2>&1 | tail -1
run() { v=$(env "$@" timeout 150 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-baseline --rope off --bits 4 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['per_kernel_ms']['palu_latent_score_tc']*1e3,1))"); echo "$*: $v"; }
for rep in 1 2; do
  run PALU_LQ_STAGES=3 PALU_LQ_RAW=6
  run X=1
  run PALU_LQ_RAW=8
  run PALU_LIB_PATH=abtmp/pf0/libpalu_b200.so
  run PALU_LIB_PATH=abtmp/pf0/libpalu_b200.so PALU_LQ_STAGES=3
done 2>&1 | tee gpurun_out/r2_lsq4.txt
