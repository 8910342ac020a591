#!/bin/bash
# round-2 final evidence: full GPU suite (long-context parity logged), bench lines, launch list, ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
rm -f gpurun_out/r02_parity_final.jsonl
PALU_PARITY_LOG=gpurun_out/r02_parity_final.jsonl timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -6 > gpurun_out/r02_pytest_gpu.txt
cat gpurun_out/r02_pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r2_fin_default.log 2>&1; tail -1 gpurun_out/r2_fin_default.log > gpurun_out/r2_fin_default.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_fin_reference.log 2>&1; tail -1 gpurun_out/r2_fin_reference.log > gpurun_out/r2_fin_reference.json
for v in "preset:--rank-k 128 --rank-v 384" "preset_k16v4:--rank-k 128 --rank-v 384 --bits 16,4" "int4:--bits 4" "int2:--bits 2" "norope:--rope off" "norope_int4:--rope off --bits 4" "norope_int2:--rope off --bits 2" "ctx16k:--context 16384" "ctx4k:--context 4096" "b4_16k:--batch 4 --context 16384" "plan_k16v4:--rank-plan kv25-75 --bits 16,4" "gqa_32k:--kv-heads 8 --context 32768"; do
  name=${v%%:*}; args=${v#*:}
  timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e $args > gpurun_out/r2_fin_$name.log 2>&1
  tail -1 gpurun_out/r2_fin_$name.log > gpurun_out/r2_fin_$name.json
  python -c "import json; d=json.load(open('gpurun_out/r2_fin_$name.json')); print('$name', round(d['value'],1), 'us; vs flashinfer', round(d.get('speedup_vs_flashinfer_step') or 0, 3))" 2>/dev/null || echo "$name failed"
done
SKIP=100 COUNT=200 bash tools/launch_list.sh > gpurun_out/r2_launch_summary.txt 2>&1; cat gpurun_out/r2_launch_summary.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"rope_score_tc_kernel|value_tc_kernel|gemv_stream|append_absorb" -c 5 -o gpurun_out/prof_r02f_default python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"rope_score_tc_kernel|value_q_kernel" -c 2 -o gpurun_out/prof_r02f_k16v4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 2 --rank-k 128 --rank-v 384 --bits 16,4 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"latent_score_q|value_q_kernel" -c 2 -o gpurun_out/prof_r02f_norope_int4 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 2 --rope off --bits 4 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
