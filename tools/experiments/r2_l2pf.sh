#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
for a in "" "--rank-k 128 --rank-v 384 --bits 16,4" "--bits 4"; do
  for rep in 1 2; do
    for e in "PALU_L2PF=0" "PALU_L2PF=1"; do
      v=$(env $e timeout 150 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-baseline $a 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})")
      echo "[$e] $a: $v"
    done
  done
done 2>&1 | tee gpurun_out/r2_l2pf.txt
