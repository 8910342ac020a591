timeout 200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tcgen05_score or medium or c1 or quantized_keys or fused" 2>&1 | tail -2
for rk in 128 256; do echo "== rank_k $rk"; timeout 120 python tools/score_trace.py --rank-k $rk --rank-v 256 2>&1 | grep -E "rope_score|MMA loop|issue span us|wake|idle"; done
for v in "default:" "k16v4:--rank-k 128 --rank-v 384 --bits 16,4" "preset:--rank-k 128 --rank-v 384" "int4:--bits 4"; do
  name=${v%%:*}; args=${v#*:}
  timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_el_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_el_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>/dev/null || echo "$name failed"
done
