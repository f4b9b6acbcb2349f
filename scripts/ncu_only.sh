#!/bin/bash
# the two ncu passes of scripts/sweep_n1.sh alone
O=gpurun_out/sweep; mkdir -p $O
export LBBSP_BENCH_NO_C3=1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:gemm_bf16_tc_kernel<\(int\)128, \(bool\)0" --launch-skip 100 -c 1 -o $O/c2_fwd_gemm \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/status
cat $O/status
cat $O/status
