# value-kernel bottleneck probe: 0 normal, 1 no MMAs (stages released on arrival), 3 no MMAs + P not gating
for m in 0 1 3; do PALU_VALUE_DIAG=$m timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"value_tc_kernel" -c 2 python tools/fused_trace.py --score-kernel tcgen05 2>&1 | grep -E "gpu__time" | tail -1 | sed "s/^/diag $m /"; done
