for cfg in "" "--rank-k 128 --rank-v 384"; do for pf in 3 0 1 6 3; do
v=$(PALU_TC_PF=$pf timeout 100 python bench.py --steps 30 --warmup 5 $cfg 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['per_kernel_ms'].get('palu_rope_score_tc',0)*1e3,1))")
echo "cfg[$cfg] pf $pf: $v"; done; done
