#!/bin/bash
# torchrun --no-python ... bash scripts/ncu_rank0.sh SCRIPT [ARGS]: rank 0 runs
# under ncu (NVLink + DRAM counters of the peer-exchange kernels), the other
# ranks run plainly. Profiling-only: replays re-bump the peers' arrival
# counters, so the run's numbers are not results.
if [ "$LOCAL_RANK" = "0" ]; then
  exec ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k "regex:peer_grad_push|peer_grad_apply|peer_speed" --launch-skip 20 -c 6 --csv \
    --log-file gpurun_out/r02_nvlink_ncu.csv python "$@"
else
  exec python "$@"
fi
