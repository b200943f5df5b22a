#!/bin/bash
# Final round check in one gpurun call: build, the whole GPU suite, smoke, the headline bench lines.
#   ROUND_DIR=r02h bash scripts/gpu_final.sh   (writes gpurun_out/$ROUND_DIR)
O=gpurun_out/${ROUND_DIR:-final}
mkdir -p $O
make -j8 all > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log; tail -4 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json
timeout 600 python bench.py --workload c3a --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c3a.json 2> $O/bench_c3a.err
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err; tail -c 300 $O/bench_c5.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
