#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "norope" 2>&1 | tail -3
PALU_PARITY_LOG=gpurun_out/r02_parity_lsq.jsonl timeout 600 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -x -k "norope" 2>&1 | tail -3
cat gpurun_out/r02_parity_lsq.jsonl | cut -c1-250
for v in "norope_int4:--rope off --bits 4" "norope_int2:--rope off --bits 2" "norope_int8:--rope off --bits 8"; do
  name=${v%%:*}; args=${v#*:}
  for lib in abtmp/prev/libpalu_b200.so paper_2407_21118_b200/libpalu_b200.so; do
    PALU_LIB_PATH=$lib timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_lsq_$name.log 2>&1
    tail -1 gpurun_out/r2_lsq_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name $lib', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>/dev/null || { echo "$name failed"; tail -3 gpurun_out/r2_lsq_$name.log; }
  done
done
