mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "medium or c1 or small or tcgen05_score" > gpurun_out/r2_gemv_tests.log 2>&1; tail -2 gpurun_out/r2_gemv_tests.log
for e in "PALU_GEMV=warp" "X=1"; do
  env $e timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-baseline > gpurun_out/r2_gemv_$e.log 2>&1
  tail -1 gpurun_out/r2_gemv_$e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"value_q_kernel|gemv_stream" -c 3 -o gpurun_out/prof_r02_vq python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 2 --rank-k 128 --rank-v 384 --bits 16,4 > gpurun_out/ncu_vq.log 2>&1; tail -2 gpurun_out/ncu_vq.log
