# rope-off latent-score kernel: stage-count sweep (ncu duration + DRAM throughput)
for st in ${STAGES:-4 8 10 12}; do
  PALU_LS_STAGES=$st timeout 300 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:"latent_score_tc|value_tc_kernel" -c 4 \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 2 --rope off 2>&1 | \
    grep -E "latent_score_tc|value_tc|gpu__time|dram__" | paste - - - | awk -v s=$st '{print "stages", s, $1, $(NF-4), $(NF)}' | sort | uniq | head -4
done
