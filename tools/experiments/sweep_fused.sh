# fused-kernel split sweep (score SMs) at the bench workload, 8 layers
run() { env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 8 --score-kernel fused $EXTRA 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$* $EXTRA', 'step_us', round(d['value'],1), r['kernel'], round(r['kernel_ms']*1e3,1))"; }
for n in ${SMS:-0 112 120 126 132}; do run PALU_SCORE_SMS=$n; done
