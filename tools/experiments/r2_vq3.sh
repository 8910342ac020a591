timeout 200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "quantized_keys" 2>&1 | tail -2
export PALU_PARITY_LOG=gpurun_out/r02_parity_vq3.jsonl; rm -f $PALU_PARITY_LOG
timeout 400 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -k "int4had or int2had or int8 or k16v" 2>&1 | tail -2
python -c "
import json
for l in open('gpurun_out/r02_parity_vq3.jsonl'): d=json.loads(l); print(d['case'], d['rel_l2'])"
timeout 120 python tools/vq_trace.py --ctas 0 --bits 16,4 --rank-k 128 --rank-v 384 2>&1 | sed "s/np.float64(\([-0-9.]*\))/\1/g" | cut -c1-200 | head -16
for v in "k16v4:--rank-k 128 --rank-v 384 --bits 16,4" "int4:--bits 4"; do
  name=${v%%:*}; args=${v#*:}
  timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_vq3_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_vq3_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>/dev/null || echo "$name failed"
done
