# GQA reconstruct-once score: L2 prefetch distance sweep (items)
for pf in 0 2 4 8; do
  v=$(PALU_TC_PF=$pf timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-baseline --kv-heads 8 --context 32768 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['per_kernel_ms']['palu_rope_score_tc']*1e3,1))")
  echo "pf $pf: $v"
done
