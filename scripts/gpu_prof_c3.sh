#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || exit 1
for w in c3c c3a; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist16 -s 2 -c 1 -o gpurun_out/hist_$w -f python bench.py --workload $w --steps 1 --warmup 2 --no-verify --no-cpu-baseline --no-e2e > gpurun_out/ncu_$w.log 2>&1
done
