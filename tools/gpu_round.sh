# round-end style evidence run: tests, smoke, default bench, variants, launch list
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-baseline --rank-k 128 --rank-v 384 > gpurun_out/bench_preset.log 2>&1; tail -1 gpurun_out/bench_preset.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-baseline --bits 4 --layers 8 > gpurun_out/bench_int4.log 2>&1; tail -1 gpurun_out/bench_int4.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-baseline --bits 2 --layers 8 > gpurun_out/bench_int2.log 2>&1; tail -1 gpurun_out/bench_int2.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-baseline --layers 4 > /dev/null 2>&1; wc -l gpurun_out/launches.csv
