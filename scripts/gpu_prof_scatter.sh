#!/bin/bash
# ncu --set full (with source) of the two MSD k_scatter launches of one c5 sort.
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
B="python bench.py --workload c5 --steps 1 --warmup 1 --no-verify --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scatter -s 0 -c 2 -o gpurun_out/scatter_full -f $B > gpurun_out/ncu_scatter.log 2>&1
tail -n 2 gpurun_out/ncu_scatter.log
