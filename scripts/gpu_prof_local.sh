#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || exit 1
B="python bench.py --workload c5 --steps 1 --warmup 1 --no-verify --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_sort -s 0 -c 1 -o gpurun_out/local_full -f $B > gpurun_out/ncu_local.log 2>&1
tail -n 2 gpurun_out/ncu_local.log
