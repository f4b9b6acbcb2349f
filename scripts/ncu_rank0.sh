#!/bin/bash
# torchrun --no-python ... bash scripts/ncu_rank0.sh SCRIPT [ARGS]: rank 0 runs
# under ncu (NVLink + DRAM counters of the kernels matching $NCU_K, default the
# peer-exchange kernels), the other ranks run plainly. Output: $NCU_OUT.
# Profiling-only: replays re-bump the peers' arrival counters, so the run's
# numbers are not results.
K=${NCU_K:-"regex:peer_grad_push|peer_grad_apply|peer_speed"}
OUT=${NCU_OUT:-gpurun_out/r02_nvlink_ncu.csv}
if [ "$LOCAL_RANK" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k "$K" --launch-skip ${NCU_SKIP:-20} -c ${NCU_COUNT:-6} --csv --log-file "$OUT" python "$@"
else
  exec python "$@"
fi
