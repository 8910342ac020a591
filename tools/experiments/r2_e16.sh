# 16-warp score epilogue (PALU_SCORE_EPI_WARPS=16) vs the 8-warp build: parity, then step A/B
mkdir -p gpurun_out
PALU_LIB_PATH=abtmp/e16/libpalu_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
A="PALU_LIB_PATH=paper_2407_21118_b200/libpalu_b200.so"; B="PALU_LIB_PATH=abtmp/e16/libpalu_b200.so"
bash tools/ab_env.sh "$A" "$B" --no-cpu --no-e2e --no-baseline --rank-k 128 --rank-v 384 --bits 16,4
bash tools/ab_env.sh "$A" "$B" --no-cpu --no-e2e --no-baseline
bash tools/ab_env.sh "$A" "$B" --no-cpu --no-e2e --no-baseline --bits 4
bash tools/ab_env.sh "$A" "$B" --no-cpu --no-e2e --no-baseline --rank-plan kv25-75 --bits 16,4
