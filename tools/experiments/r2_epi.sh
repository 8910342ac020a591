#!/bin/bash
# score epilogue: parity subset, per-unit trace (diagnostic build), bench A/B
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
TAG=${1:-x}
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "quantized_keys or fused or medium or c1 or tcgen05_score" 2>&1 | tail -2
for rk in 128 256; do
  PALU_LIB_PATH=abtmp/diag/libpalu_b200.so PALU_SCORE_TRACE=1 timeout 300 python tools/score_trace.py --rank-k $rk --rank-v 256 > gpurun_out/score_trace_${TAG}_r$rk.txt 2>&1
  sed -n 1,12p gpurun_out/score_trace_${TAG}_r$rk.txt
done
for v in "default:" "preset:--rank-k 128 --rank-v 384" "int4:--bits 4" "k16v4:--rank-k 128 --rank-v 384 --bits 16,4"; do
  name=${v%%:*}; args=${v#*:}
  timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_${TAG}_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_${TAG}_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>/dev/null || echo "$name failed"
done
