#!/bin/bash
# Round evidence in one gpurun call: GPU tests, smoke, bench lines for every
# config, ncu launch lists, and ncu --set full captures of the top kernels.
#   ROUND_DIR=r02a bash scripts/gpu_profile_round.sh   (writes gpurun_out/$ROUND_DIR)
O=gpurun_out/${ROUND_DIR:-round}
mkdir -p $O
make -j8 all > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 400 $O/bench_c2.json
for w in c1 c3a c3b c3c c3d; do timeout 600 python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python bench.py --workload c5 --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err; tail -c 300 $O/bench_c5.json
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c4_1gpu.json 2> $O/bench_c4.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.json 2> $O/bench_reference.err
rm -f scripts/microbench/variants/*.so
# N>1 plumbing on the one GPU of the box (two ranks share it; gloo for the host collectives): every field of the N>1 line
FS_BENCH_SHARE_GPU=1 FS_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_n2_shared.json 2> $O/bench_n2_shared.err; tail -c 600 $O/bench_n2_shared.json
timeout 600 python scripts/microbench/wide_skew.py $((1 << 29)) > $O/wide_skew_c5size.txt 2>&1
NB="--no-e2e --no-cpu-baseline --no-verify"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 5 --warmup 3 $NB > $O/ncu_launch_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv python bench.py --workload c5 --steps 2 --warmup 1 $NB > $O/ncu_launch_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hist16|k_expand16" -s 4 -c 2 -o $O/prof_c2 -f python bench.py --steps 3 --warmup 3 $NB > $O/ncu_full_c2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_top16_hist|k_scatter|k_local_sort" -c 5 -o $O/prof_c5 -f python bench.py --workload c5 --steps 1 --warmup 0 $NB > $O/ncu_full_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hist16" -s 3 -c 1 -o $O/prof_c3a -f python bench.py --workload c3a --steps 2 --warmup 3 $NB > $O/ncu_full_c3a.log 2>&1
ls -la $O
