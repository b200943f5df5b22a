#!/bin/bash
# ncu --set full of one c5 sort's level-1 k_scatter and one k_local_sort launch.
mkdir -p gpurun_out/r02d
make -j8 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
B="python bench.py --workload c5 --steps 1 --warmup 1 --no-verify --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_local_sort" -s 0 -c 3 -o gpurun_out/r02d/c5kern -f $B > gpurun_out/r02d/ncu_c5kern.log 2>&1
tail -n 2 gpurun_out/r02d/ncu_c5kern.log
