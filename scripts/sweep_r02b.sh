#!/bin/bash
# Round-2 one-GPU sweep after the pair kernel (gpurun_out/r02b/): bench (C2
# default) + reference arm, smoke, ncu launch list of the bench command, ncu
# --set full of the pair worker kernel.
O=${OUT:-gpurun_out/r02b}; mkdir -p $O
st() { echo "$1 rc=$2" >> $O/status; }
timeout 900 python bench.py --steps 20 --warmup 5 > $O/c2_n1.json 2> $O/c2_n1.err; st bench $?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/ref_n1.json 2> $O/ref_n1.err; st ref $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; st smoke $?
export LBBSP_BENCH_NO_C3=1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1500 -c 300 --csv \
  --log-file $O/c2_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/ncu_list.log 2>&1; st ncu_list $?
unset LBBSP_BENCH_NO_C3
NO_STRAGGLE=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:c2_pair --launch-skip 3 -c 1 \
  -o $O/c2_pair python scripts/sanitize_c2.py > $O/ncu_pair.log 2>&1; st ncu_pair $?
cat $O/status
