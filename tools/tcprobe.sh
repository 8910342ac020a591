# tcgen05 score-kernel pipeline probe (profiling modes are env-selected, off by default)
run() { env "$@" timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e --layers 8 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', 'score_us', round(d['roofline']['kernel_ms']*1e3,1))"; }
for m in 0 1 2 3 4 5 6 7; do run PALU_TC_PROFILE_MODE=$m PALU_TC_PF=0; done
