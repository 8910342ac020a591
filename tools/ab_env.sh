# usage: bash tools/ab_env.sh "ENV_A" "ENV_B" [bench args]  -- interleaved A/B of bench.py step time
A="$1"; B="$2"; shift 2
for e in "$A" "$B" "$A" "$B"; do
  v=$(env $e timeout 100 python bench.py --steps 30 --warmup 5 "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['per_kernel_ms'].get('palu_rope_score_tc',0)*1e3,1))")
  echo "[$e] $*: $v"
done
