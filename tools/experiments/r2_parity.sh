mkdir -p gpurun_out
export PALU_PARITY_LOG=gpurun_out/r02_parity.jsonl
rm -f $PALU_PARITY_LOG
timeout 900 python -m pytest tests/test_gpu_long_parity.py -q -m gpu > gpurun_out/r2_long_parity.log 2>&1; tail -3 gpurun_out/r2_long_parity.log
timeout 600 python -m pytest tests -x -q -m gpu --deselect tests/test_gpu_long_parity.py > gpurun_out/r2_pytest_gpu.log 2>&1; tail -1 gpurun_out/r2_pytest_gpu.log
nproc > gpurun_out/r2_host.txt; lscpu | head -20 >> gpurun_out/r2_host.txt; free -g >> gpurun_out/r2_host.txt
