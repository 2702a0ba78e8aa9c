R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/q2
timeout 300 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/q2/b2.json 2> gpurun_out/q2/b2.err
timeout 300 $R --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 --update sharded --no-cpu-baseline > gpurun_out/q2/b2s.json 2> gpurun_out/q2/b2s.err
for u in replicated sharded none; do
  timeout 300 $R --nproc-per-node 2 --master-port 29603 tools/ar_call.py --update $u > gpurun_out/q2/call_$u.json 2>&1
done
timeout 300 $R --nproc-per-node 2 --master-port 29604 tools/ar_call.py --update none --elems 268435456 > gpurun_out/q2/call_1g.json 2>&1
MASTER_PORT=29711 bash tools/ncu_rank0.sh 2 gpurun_out/q2/ncu_repl.csv allreduce tools/ar_call.py --update replicated > gpurun_out/q2/ncu_repl.log 2>&1
MASTER_PORT=29712 bash tools/ncu_rank0.sh 2 gpurun_out/q2/ncu_shard.csv allreduce tools/ar_call.py --update sharded > gpurun_out/q2/ncu_shard.log 2>&1
MASTER_PORT=29713 bash tools/ncu_rank0.sh 2 gpurun_out/q2/ncu_1g.csv allreduce tools/ar_call.py --update none --elems 268435456 > gpurun_out/q2/ncu_1g.log 2>&1
timeout 300 ./tools/nvls_probe 256 10 > gpurun_out/q2/nvls.txt 2>&1
MD_AR_SYS_FENCE=1 timeout 400 $R --nproc-per-node 2 --master-port 29605 tools/stress_fused.py --calls 500 --route tree > gpurun_out/q2/st_tree_sys.json 2> gpurun_out/q2/st_tree_sys.err
timeout 400 $R --nproc-per-node 2 --master-port 29606 tools/stress_fused.py --calls 500 --route tree > gpurun_out/q2/st_tree.json 2> gpurun_out/q2/st_tree.err
