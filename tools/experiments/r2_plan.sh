timeout 300 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_long_parity.py 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --rank-plan kv25-75 > gpurun_out/r2_bench_plan.log 2>&1
tail -1 gpurun_out/r2_bench_plan.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('plan', d['config']['workload'], round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()}, d.get('speedup_vs_flashinfer_step'))" 2>&1 | tail -2
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline --rank-plan kv25-75 --bits 16,4 > gpurun_out/r2_bench_plan_k16v4.log 2>&1
tail -1 gpurun_out/r2_bench_plan_k16v4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('plan k16v4', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>&1 | tail -2
