# tcgen05 score-kernel pipeline probe (profiling modes are env-selected, off by default):
# 1 epilogue skips math, 2 MMA skips TMA waits, 4 MMA skips TMEM-empty waits
run() { env "$@" timeout 120 python bench.py --steps 5 --warmup 2 --no-cpu --no-e2e --no-baseline --layers 8 $EXTRA 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$* $EXTRA', 'score_us', round(d['roofline']['kernel_ms']*1e3,1))"; }
for m in ${MODES:-0 1}; do run PALU_TC_PROFILE_MODE=$m; done
