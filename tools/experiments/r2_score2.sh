echo "== UH=1 r128"; PALU_SCORE_UH=1 timeout 120 python tools/score_trace.py --rank-k 128 --rank-v 256 2>&1 | grep -E "rope_score|MMA loop|issue span us|wake|idle"
for e in "PALU_SCORE_UH=1" "PALU_SCORE_UH=2"; do
for v in "k16v4:--rank-k 128 --rank-v 384 --bits 16,4"; do
  name=${v%%:*}; args=${v#*:}
  env $e timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline $args > gpurun_out/r2_bench_uh_$name.log 2>&1
  tail -1 gpurun_out/r2_bench_uh_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e $name', round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})" 2>/dev/null || echo "$name failed"
done; done
