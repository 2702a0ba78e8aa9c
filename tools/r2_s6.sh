R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s6; mkdir -p $O
# NVLink bytes of the allreduce kernels on rank 0 of a live job
MASTER_PORT=29731 bash tools/ncu_rank0.sh 2 $O/ncu_n2_sharded.csv allreduce tools/ar_call.py --update sharded > $O/ncu_n2_sharded.log 2>&1
MASTER_PORT=29732 bash tools/ncu_rank0.sh 2 $O/ncu_n2_repl.csv allreduce tools/ar_call.py --update replicated > $O/ncu_n2_repl.log 2>&1
MASTER_PORT=29733 bash tools/ncu_rank0.sh 2 $O/ncu_n2_1g.csv allreduce tools/ar_call.py --update none --elems 268435456 > $O/ncu_n2_1g.log 2>&1
MASTER_PORT=29734 bash tools/ncu_rank0.sh 4 $O/ncu_n4_sharded.csv allreduce tools/ar_call.py --update sharded > $O/ncu_n4_sharded.log 2>&1
MASTER_PORT=29735 bash tools/ncu_rank0.sh 4 $O/ncu_n4_repl.csv allreduce tools/ar_call.py --update replicated > $O/ncu_n4_repl.log 2>&1
MASTER_PORT=29736 bash tools/ncu_rank0.sh 4 $O/ncu_n4_1g.csv allreduce tools/ar_call.py --update none --elems 268435456 > $O/ncu_n4_1g.log 2>&1
for n in 2 4; do
  timeout 200 $R --nproc-per-node $n --master-port 29609 tools/ar_call.py --update none --elems 268435456 --calls 8 > $O/call_n${n}_1g.json 2>&1
done
timeout 400 python bench.py > $O/b1.json 2> $O/b1.err
timeout 400 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > $O/b2.json 2> $O/b2.err
timeout 400 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > $O/b4.json 2> $O/b4.err
timeout 400 python bench.py --impl reference > $O/r1.json 2> $O/r1.err
timeout 400 $R --nproc-per-node 2 --master-port 29603 bench.py --impl reference --gpus 2 > $O/r2.json 2> $O/r2.err
timeout 400 $R --nproc-per-node 4 --master-port 29604 bench.py --impl reference --gpus 4 > $O/r4.json 2> $O/r4.err
timeout 600 $R --nproc-per-node 1 --master-port 29605 bench_dimd.py > $O/d1.json 2> $O/d1.err
timeout 600 $R --nproc-per-node 2 --master-port 29606 bench_dimd.py > $O/d2.json 2> $O/d2.err
MD_BENCH_NOCLOCK=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
MD_BENCH_NOCLOCK=1 ncu --set full --clock-control none --import-source on -k regex:sgd_vec_kernel \
  -s 3 -c 1 -o $O/update_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
