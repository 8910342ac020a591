# round evidence run: tests, smoke, default bench, variants, launch list, ncu captures
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | cut -c1-300
for v in "preset:--rank-k 128 --rank-v 384" "preset_k16v4:--rank-k 128 --rank-v 384 --bits 16,4" "int4:--bits 4" "norope:--rope off" "norope_int4:--rope off --bits 4" "ctx16k:--context 16384" "ctx4k:--context 4096" "b4_16k:--batch 4 --context 16384"; do
  name=${v%%:*}; args=${v#*:}
  timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e $args > gpurun_out/bench_$name.log 2>&1
  tail -1 gpurun_out/bench_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); u=d.get('uncompressed') or {}; print('$name', round(d['value'],1), 'us/step; vs best uncompressed', round(u.get('palu_speedup_vs_best_est', 0), 3))"
done
SKIP=100 COUNT=200 bash tools/launch_list.sh > gpurun_out/launch_summary.txt 2>&1; cat gpurun_out/launch_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rope_score_tc_kernel|value_tc_kernel|latent_score_tc" -c 3 -o gpurun_out/prof_r01_final python tools/fused_trace.py --score-kernel tcgen05 > gpurun_out/ncu_final.log 2>&1; tail -1 gpurun_out/ncu_final.log
timeout 300 ncu --set full --clock-control none -k regex:"latent_score_tc" -c 1 -o gpurun_out/prof_r01_norope python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 2 --rope off > /dev/null 2>&1; ls gpurun_out/*.ncu-rep
