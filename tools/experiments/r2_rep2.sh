mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_long_parity.py -q -m gpu -x -p no:cacheprovider -k "gqa" 2>&1 | tail -2
bash tools/ab_env.sh "PALU_GQA_REP=0" "PALU_GQA_REP=1" --no-cpu --no-e2e --no-baseline --kv-heads 8 --context 32768
PALU_LIB_PATH=abtmp/tr/libpalu_b200.so timeout 300 python tools/score_trace.py --kv-heads 8 --context 32768 --rank-k 64 --rank-v 64 2>&1 | tail -18
