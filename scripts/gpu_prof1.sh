#!/bin/bash
# hist16 phase trace + ncu full capture of one onesweep pass (c5) and of the digit histogram.
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || exit 1
./scripts/microbench/ht > gpurun_out/hist_trace.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 2 -c 1 \
  -o gpurun_out/onesweep_full -f python bench.py --workload c5 --steps 1 --warmup 1 --no-verify --no-cpu-baseline --no-e2e > gpurun_out/ncu_onesweep.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_digit_hist -c 1 \
  -o gpurun_out/digithist_full -f python bench.py --workload c5 --steps 1 --warmup 1 --no-verify --no-cpu-baseline --no-e2e > gpurun_out/ncu_digithist.log 2>&1
tail -3 gpurun_out/ncu_onesweep.log gpurun_out/ncu_digithist.log
head -30 gpurun_out/hist_trace.log
