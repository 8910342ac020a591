timeout 300 python tools/fused_trace.py --score-kernel tcgen05 2>&1 | grep -E "rope_attend|palu_value|value:|phases" | head -4 | cut -c1-300
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"value_tc_kernel|value_merge" -c 4 python tools/fused_trace.py --score-kernel tcgen05 2>&1 | grep -E "value_tc_kernel|value_merge|gpu__time_duration" | head -12
