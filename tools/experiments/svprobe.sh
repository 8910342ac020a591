run() { env "$@" timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e --layers 8 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', 'sv_us', round(d['roofline']['per_kernel_ms']['palu_softmax_value']*1e3,1))"; }
for c in 18 37 74 111 148 296; do run PALU_SV_CHUNKS=$c; done
