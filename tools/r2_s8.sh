R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s8; mkdir -p $O
for n in 2 4; do
  MD_AR_TRACE=1 timeout 200 $R --nproc-per-node $n --master-port 29641 tools/trace_push.py > $O/trace_n${n}_sharded.json 2> $O/trace_n${n}_sharded.err
done
timeout 400 python bench.py > $O/b1.json 2> $O/b1.err
MD_DIMD_TIMING=1 timeout 600 $R --nproc-per-node 4 --master-port 29607 bench_dimd.py --cpu-records 0 --epochs 5 > $O/d4_timing.json 2> $O/d4_timing.err
