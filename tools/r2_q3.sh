R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/q3; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dimd.py tests/test_gpu_misc.py -q -x 2>&1 | tail -15 > $O/pytest_dimd.txt
for x in push pull; do
  timeout 400 $R --nproc-per-node 2 --master-port 29607 bench_dimd.py --exchange $x --cpu-records 0 > $O/d2_$x.json 2> $O/d2_$x.err
done
MASTER_PORT=29711 bash tools/ncu_rank0.sh 2 $O/ncu_shard.csv allreduce tools/ar_call.py --update sharded > $O/ncu_shard.log 2>&1
MASTER_PORT=29712 bash tools/ncu_rank0.sh 2 $O/ncu_repl.csv allreduce tools/ar_call.py --update replicated > $O/ncu_repl.log 2>&1
MASTER_PORT=29713 bash tools/ncu_rank0.sh 2 $O/ncu_1g.csv allreduce tools/ar_call.py --update none --elems 268435456 > $O/ncu_1g.log 2>&1
