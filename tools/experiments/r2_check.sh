mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_long_parity.py > gpurun_out/r2_pytest_gpu.log 2>&1; tail -1 gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_bench_default.log 2>&1; tail -1 gpurun_out/r2_bench_default.log | cut -c1-3000
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --rank-k 128 --rank-v 384 --bits 16,4 > gpurun_out/r2_bench_k16v4.log 2>&1; tail -1 gpurun_out/r2_bench_k16v4.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.log 2>&1; tail -1 gpurun_out/r2_bench_ref.log
