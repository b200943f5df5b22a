#!/bin/bash
# quick check: u16 GPU tests, hist trace, c2 bench
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_u16.py -x -q > gpurun_out/pytest_u16.log 2>&1; tail -3 gpurun_out/pytest_u16.log
./scripts/microbench/ht > gpurun_out/hist_trace.log 2>&1; sed -n '/rep 3/,/scan end/p' gpurun_out/hist_trace.log
for i in 1 2; do timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c2_q$i.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bench_c2_q$i.json'));print(d['ms_per_step'],d['phases_ms'],d['roofline']['frac'])"; done
