mkdir -p gpurun_out
export PALU_PARITY_LOG=gpurun_out/r02_parity_vq.jsonl
rm -f $PALU_PARITY_LOG
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "quantized_keys" -x > gpurun_out/r2_vq_tests.log 2>&1; tail -3 gpurun_out/r2_vq_tests.log
timeout 600 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -k "int4had or int2had or int8 or k16v" > gpurun_out/r2_vq_long.log 2>&1; tail -3 gpurun_out/r2_vq_long.log
for v in "k16v4:--rank-k 128 --rank-v 384 --bits 16,4" "int4:--bits 4" "k16v2:--rank-k 128 --rank-v 384 --bits 16,2" "int8:--bits 8"; do
  name=${v%%:*}; args=${v#*:}
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_vq_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_vq_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()}, 'value GB/s', round(d['roofline']['value_hbm_gbs'] or 0))"
done
