timeout 120 python tools/vq_trace.py --ctas 0 2>&1 | sed 's/np.float64(\([-0-9.]*\))/\1/g' | cut -c1-300
timeout 180 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "quantized_keys or fused_attend or c1 or medium" 2>&1 | tail -2
for v in "default:" "k16v4:--rank-k 128 --rank-v 384 --bits 16,4" "int4:--bits 4" "preset:--rank-k 128 --rank-v 384"; do
  name=${v%%:*}; args=${v#*:}
  timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_vq_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_vq_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()}, 'value GB/s', round(d['roofline']['value_hbm_gbs'] or 0))" 2>/dev/null || echo "$name failed"
done
