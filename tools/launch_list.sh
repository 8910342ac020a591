# steady-state launch list of one bench step (our kernels only, after warm-up)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"gemv|append|absorb|rope_score|value_tc|value_q|value_merge|softmax_value|advance|rope_attend" \
  -s ${SKIP:-300} -c ${COUNT:-300} --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-baseline --layers ${LAYERS:-8} $EXTRA > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
