mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2_pytest_gpu.log 2>&1; tail -1 gpurun_out/r2_pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/r2_bench_default.log 2>&1; tail -1 gpurun_out/r2_bench_default.log | cut -c1-600
for v in "preset:--rank-k 128 --rank-v 384" "preset_k16v4:--rank-k 128 --rank-v 384 --bits 16,4" "int4:--bits 4"; do
  name=${v%%:*}; args=${v#*:}
  timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e $args > gpurun_out/r2_bench_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_$name.log | cut -c1-400
done
