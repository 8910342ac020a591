#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
run() { v=$(env "$@" timeout 150 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['per_kernel_ms']['palu_value_tc']*1e3,1))"); echo "$*: $v"; }
for rep in 1 2; do
  run X=1
  run PALU_LIB_PATH=abtmp/vh4/libpalu_b200.so
  run PALU_LIB_PATH=abtmp/vh99/libpalu_b200.so
done 2>&1 | tee gpurun_out/r2_vhead.txt
