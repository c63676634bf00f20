#!/bin/bash
# One GPU session that produces everything profiles/ holds for a round (run under gpurun).
set -x
mkdir -p gpurun_out/prof
timeout 400 python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/prof/bench_reference.json 2>&1
timeout 300 python bench.py --config cfg3 --steps 20 --no-cpu-baseline > gpurun_out/prof/bench_cfg3.json 2>&1
timeout 300 python bench.py --config cfg4 --steps 20 > gpurun_out/prof/bench_cfg4.json 2>&1
timeout 300 python bench.py --config cfg4 --simulate-world 8 --steps 10 > gpurun_out/prof/bench_cfg4_sim8.json 2>&1
timeout 300 python bench.py --sharded --steps 20 --no-cpu-baseline > gpurun_out/prof/bench_sharded1.json 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches.csv \
  python bench.py --steps 2 --warmup 3 --profile --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -s 16 -c 9 -o gpurun_out/prof/full \
  python bench.py --steps 2 --warmup 3 --profile --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/prof
timeout 300 python bench.py --config cfg5 --steps 5 --warmup 2 > gpurun_out/prof/bench_cfg5.json 2>&1
timeout 300 python bench.py --config cfg5 --impl reference > gpurun_out/prof/bench_cfg5_reference.json 2>&1
timeout 300 ncu --set full --clock-control none -k regex:replay -c 1 -o gpurun_out/prof/replay python bench.py --config cfg5 --steps 1 --warmup 0 > /dev/null 2>&1
ls -la gpurun_out/prof
