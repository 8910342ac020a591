#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"latent_score_q|value_q_kernel" -c 2 -o gpurun_out/prof_lsq python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 2 --rope off --bits 4 > /dev/null 2>&1
python profiles/ncu_summary.py gpurun_out/prof_lsq.ncu-rep > gpurun_out/prof_lsq.txt 2>&1
ncu -i gpurun_out/prof_lsq.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
keys=[k for k in h if any(s in k for s in ['l1tex__data_pipe_lsu_wavefronts_mem_shared','smsp__sass_inst_executed_op_shared','l1tex__data_bank_conflicts_pipe_lsu_mem_shared','sm__memory_throughput','l1tex__throughput','smsp__inst_executed.sum','sm__pipe_shared_cycles','lts__t_bytes.sum'])]
for r in rows[2:]:
    print(r[h.index('Kernel Name')][:60])
    for k in keys: print('  ',k, r[h.index(k)])
" >> gpurun_out/prof_lsq.txt
