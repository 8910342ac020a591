set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.log 2>&1; tail -2 gpurun_out/bench_default.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline --score-kernel tcgen05 > gpurun_out/bench_tc.log 2>&1; tail -1 gpurun_out/bench_tc.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline --rank-k 128 --rank-v 384 > gpurun_out/bench_preset.log 2>&1; tail -1 gpurun_out/bench_preset.log
