#!/bin/bash
# NVLink bytes of one rank's kernels inside a live multi-GPU job: rank 0 runs
# under ncu, ranks 1..N-1 run plain. gpurun's ncu first runs the profiled
# command once WITHOUT ncu (it must exit 0) and only then under ncu, so the
# peers run the job twice, once for each of rank 0's runs. Single-pass metrics
# only: a replayed kernel would wait for peers that already finished (NVLink
# counters alone are one pass; adding gpu__time_duration makes it three).
#   tools/ncu_rank0.sh N OUT.csv KERNEL_REGEX script.py [args...]
N=$1; OUT=$2; KREGEX=$3; shift 3
export MASTER_ADDR=127.0.0.1 MASTER_PORT=${MASTER_PORT:-29710} WORLD_SIZE=$N LOCAL_WORLD_SIZE=$N
pids=()
for ((r = 1; r < N; r++)); do
  (for run in 1 2; do RANK=$r LOCAL_RANK=$r timeout 240 python "$@" > /dev/null 2>&1; done) &
  pids+=($!)
done
RANK=0 LOCAL_RANK=0 ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
  -k "regex:$KREGEX" --clock-control none --csv --log-file "$OUT" python "$@"
for p in "${pids[@]}"; do wait "$p"; done
