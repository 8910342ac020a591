timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_long_parity.py -q -m gpu -x -p no:cacheprovider -k "gqa" 2>&1 | tail -1
bash tools/ab_env.sh "PALU_LIB_PATH=abtmp/prev_rep/libpalu_b200.so" "PALU_LIB_PATH=paper_2407_21118_b200/libpalu_b200.so" --no-cpu --no-e2e --no-baseline --kv-heads 8 --context 32768
