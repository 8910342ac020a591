#!/bin/bash
# packed-key hand-off relay: parity + bench
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for v in "int4:--bits 4" "int2:--bits 2" "k4v4p:--rank-k 128 --rank-v 384 --bits 4" "norope_int4:--rope off --bits 4" "k16v4:--rank-k 128 --rank-v 384 --bits 16,4" "default:"; do
  name=${v%%:*}; args=${v#*:}
  timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_relay_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_relay_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>/dev/null || { echo "$name failed"; tail -3 gpurun_out/r2_bench_relay_$name.log; }
done
