timeout 200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gqa" 2>&1 | tail -3
export PALU_PARITY_LOG=gpurun_out/r02_parity_gqa.jsonl; rm -f $PALU_PARITY_LOG
timeout 500 python -m pytest tests/test_gpu_long_parity.py -q -m gpu -k "gqa" 2>&1 | tail -3
cat gpurun_out/r02_parity_gqa.jsonl
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --kv-heads 8 --context 32768 > gpurun_out/r2_bench_gqa.log 2>&1
tail -1 gpurun_out/r2_bench_gqa.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gqa', d['config']['workload'], round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()}, d['uncompressed'])" 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --kv-heads 8 --context 32768 --bits 16,4 > gpurun_out/r2_bench_gqa_k16v4.log 2>&1
tail -1 gpurun_out/r2_bench_gqa_k16v4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gqa k16v4', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()}, d.get('speedup_vs_flashinfer_step'))" 2>&1 | tail -2
