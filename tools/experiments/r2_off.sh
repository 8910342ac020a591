timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "offline or build_fused_gpu" -s 2>&1 | grep -E "decompose_gpu|passed|failed|Error|assert" | head
