#!/bin/bash
# Wide-path GPU tests + ncu --set full (with source) of one k_local_sort launch at c5.
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/pytest_wide.log 2>&1; tail -2 gpurun_out/pytest_wide.log
B="python bench.py --workload c5 --steps 1 --warmup 1 --no-verify --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_sort -s 0 -c 1 -o gpurun_out/local_full -f $B > gpurun_out/ncu_local.log 2>&1
tail -n 2 gpurun_out/ncu_local.log
