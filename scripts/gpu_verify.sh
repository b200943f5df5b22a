O=gpurun_out/r02g_verify; mkdir -p $O
make -j8 all > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 300 python scripts/microbench/nvls_probe.py > $O/nvls_probe.txt 2>&1; tail -5 $O/nvls_probe.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 300 $O/bench_c2.json
timeout 600 python bench.py --workload c3a --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_c3a.json 2> $O/bench_c3a.err
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err; tail -c 300 $O/bench_c5.json
