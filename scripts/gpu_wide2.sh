#!/bin/bash
mkdir -p gpurun_out
make -j8 all > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_wide.py -x -q > gpurun_out/pytest_wide.log 2>&1; tail -5 gpurun_out/pytest_wide.log
timeout 600 python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));print(d['ms_per_step'],d['phases_ms'])"
python scripts/microbench/wide_variants.py 2>&1 | tail -5
