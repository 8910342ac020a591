# fused score+value kernel vs the two-kernel path across context lengths
for ctx in 4096 16384 65536; do
  for sk in auto fused auto fused; do
    v=$(timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --no-baseline --context $ctx --score-kernel $sk 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
    echo "ctx $ctx $sk: $v"
  done
done
