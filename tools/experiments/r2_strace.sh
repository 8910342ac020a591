for rk in 128 256; do echo "== rank_k $rk"; timeout 120 python tools/score_trace.py --rank-k $rk --rank-v 256 2>&1 | tail -22; done
