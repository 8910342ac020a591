timeout 300 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_long_parity.py 2>&1 | tail -2
for v in "default:" "k16v4:--rank-k 128 --rank-v 384 --bits 16,4"; do
  name=${v%%:*}; args=${v#*:}
  timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_c2_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_c2_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>/dev/null || echo "$name failed"
done
