timeout 300 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_long_parity.py 2>&1 | tail -2
export PALU_PARITY_LOG=gpurun_out/r02_parity_vb.jsonl; rm -f $PALU_PARITY_LOG
timeout 300 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -k "r256_bf16_64k or preset_bf16" 2>&1 | tail -2
python -c "
import json
for l in open('gpurun_out/r02_parity_vb.jsonl'): d=json.loads(l); print(d['case'], d['rel_l2'], d['value_kernel'])"
for e in "PALU_VALUE_KERNEL=tc_bf16_role" "X=1"; do
for v in "default:" "preset:--rank-k 128 --rank-v 384"; do
  name=${v%%:*}; args=${v#*:}
  env $e timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_vb_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_vb_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e $name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>/dev/null || echo "$name failed"
done; done
