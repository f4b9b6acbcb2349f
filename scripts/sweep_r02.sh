#!/bin/bash
# Round-2 one-GPU measurement sweep (everything lands in gpurun_out/r02/):
# GPU tests, bench (C2 default) + reference arm, smoke, ncu launch list of the
# bench command, ncu --set full of the fused worker kernel and of the C3 dW
# GEMM, compute-sanitizer racecheck/synccheck of a C2 round.
O=gpurun_out/r02; mkdir -p $O
st() { echo "$1 rc=$2" >> $O/status; }
timeout 900 python bench.py --steps 20 --warmup 5 > $O/c2_n1.json 2> $O/c2_n1.err; st bench $?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_n1.json 2> $O/ref_n1.err; st ref $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; st smoke $?
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; st pytest $?
export LBBSP_BENCH_NO_C3=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1500 -c 300 --csv \
  --log-file $O/c2_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/ncu_list.log 2>&1; st ncu_list $?
unset LBBSP_BENCH_NO_C3
timeout 600 ncu --set full --import-source on --clock-control none -k regex:c2_fused --launch-skip 3 -c 1 \
  -o $O/c2_fused python scripts/sanitize_c2.py > $O/ncu_fused.log 2>&1; st ncu_fused $?
ROUNDS=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16_tc2 --launch-skip 8 -c 11 \
  -o $O/c3_gemms python scripts/c3_one_gpu.py > $O/ncu_c3.log 2>&1; st ncu_c3 $?
ROUNDS=3 timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis python scripts/sanitize_c2.py > $O/racecheck.log 2>&1; st racecheck $?
ROUNDS=3 timeout 900 compute-sanitizer --tool synccheck python scripts/sanitize_c2.py > $O/synccheck.log 2>&1; st synccheck $?
ROUNDS=3 timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_c2.py > $O/memcheck.log 2>&1; st memcheck $?
cat $O/status
