R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s14; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_c5.py tests/test_gpu_allreduce.py -q -x 2>&1 | tail -3 > $O/pytest.txt
for n in 2 4; do
  MD_AR_TRACE=1 timeout 200 $R --nproc-per-node $n --master-port 29641 tools/trace_push.py > $O/trace_n${n}_sharded.json 2> $O/trace_n${n}_sharded.err
  timeout 300 $R --nproc-per-node $n --master-port 29602 bench.py --gpus $n --no-cpu-baseline > $O/b$n.json 2> $O/b$n.err
  timeout 300 $R --nproc-per-node $n --master-port 29603 bench.py --gpus $n --no-cpu-baseline > $O/b${n}_again.json 2> $O/b${n}_again.err
  timeout 200 $R --nproc-per-node $n --master-port 29609 tools/ar_call.py --update none --elems 268435456 --calls 8 > $O/call_n${n}_1g.json 2>&1
  timeout 400 $R --nproc-per-node $n --master-port 29604 tools/stress_fused.py --calls 1000 --sharded > $O/st${n}_sharded.json 2> $O/st${n}_sharded.err
done
