#!/bin/bash
# compute-sanitizer over scripts/sanity_small.py (every C-ABI entry point: k_hist16,
# k_sort16_small, k_expand16, k_scan, the wide path's k_top16_hist / k_scatter /
# k_local_sort / k_tiny_bins / k_heavy, k_expand_to_peers, the trie kernels,
# the host-streamed sort) with memcheck, racecheck, synccheck and initcheck.
# Logs: $1 (default gpurun_out/r02_sanitizer).
O=${1:-gpurun_out/r02_sanitizer}
mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  [ $tool = initcheck ] && extra="--track-unused-memory no"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 7 \
      --target-processes all python scripts/sanity_small.py > $O/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $O/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanity_small" $O/$tool.log | tail -3 | tee -a $O/summary.txt
done
