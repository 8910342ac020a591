#!/bin/bash
# usage: bash tools/ab_lib.sh LIB_A LIB_B [bench args] -- interleaved A/B of two library builds
# (step time and the per-kernel times of bench.py's profile pass)
A="$1"; B="$2"; shift 2
for l in "$A" "$B" "$A" "$B"; do
  v=$(PALU_LIB_PATH=$l timeout 150 python bench.py --steps 30 --warmup 5 --no-cpu --no-e2e --no-baseline "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k: round(v*1e3,1) for k,v in d['roofline']['per_kernel_ms'].items()})")
  echo "[$l] $*: $v"
done
