# replicated-B (GQA) score: parity (golden + 32K oracle), then step A/B against the per-head path
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_long_parity.py -q -m gpu -x -p no:cacheprovider -k "gqa" 2>&1 | tail -3
cat gpurun_out/*.jsonl 2>/dev/null | tail -2
bash tools/ab_env.sh "PALU_GQA_REP=0" "PALU_GQA_REP=1" --no-cpu --no-e2e --no-baseline --kv-heads 8 --context 32768
