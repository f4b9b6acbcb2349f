#!/bin/bash
# One-GPU measurement sweep: GPU tests, default bench (C2), reference arm,
# ncu launch list of steady-state C2 rounds and one --set full capture of the
# C2 forward GEMM. Everything lands in gpurun_out/sweep/.
O=gpurun_out/sweep; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/status
timeout 900 python bench.py > $O/c2_n1.json 2> $O/c2_n1.err; echo "c2 rc=$?" >> $O/status
timeout 900 python bench.py --impl reference > $O/ref_n1.json 2> $O/ref_n1.err; echo "ref rc=$?" >> $O/status
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/status
export LBBSP_BENCH_NO_C3=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --launch-skip 900 -c 180 --csv \
  --log-file $O/c2_launches.csv python bench.py --steps 60 --warmup 3 --no-cpu-baseline > $O/ncu_list.log 2>&1; echo "ncu list rc=$?" >> $O/status
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:gemm_bf16_tc_kernel<\(int\)128, \(bool\)0" --launch-skip 100 -c 1 -o $O/c2_fwd_gemm \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/status
cat $O/status
