# A/B of the PDL split form (PALU_PDL_SPLIT=0: split kernels wait at entry) and PDL off
for cfg in "" "--rank-k 128 --rank-v 384"; do
  for env in "PALU_PDL_SPLIT=1" "PALU_PDL_SPLIT=0" "PALU_PDL=0" "PALU_PDL_SPLIT=1" "PALU_PDL_SPLIT=0"; do
    v=$(env $env timeout 300 python bench.py --steps 30 --warmup 5 $cfg 2>/dev/null | tail -1 | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))")
    echo "cfg[$cfg] $env: $v us/step"
  done
done
