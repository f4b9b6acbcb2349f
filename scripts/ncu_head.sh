#!/bin/bash
O=gpurun_out/sweep; mkdir -p $O
export LBBSP_BENCH_NO_C3=1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:head_mma_kernel<\(bool\)1>" --launch-skip 100 -c 1 -o $O/c2_head \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_head.log 2>&1; echo "ncu head rc=$?"
