R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s12; mkdir -p $O
for n in 2 4; do
  timeout 300 $R --nproc-per-node $n --master-port 29602 bench.py --gpus $n --no-cpu-baseline > $O/b$n.json 2> $O/b$n.err
  timeout 400 $R --nproc-per-node $n --master-port 29604 tools/stress_fused.py --calls 2000 --sharded > $O/st${n}_sharded.json 2> $O/st${n}_sharded.err
  timeout 400 $R --nproc-per-node $n --master-port 29605 tools/stress_fused.py --calls 2000 > $O/st${n}_auto.json 2> $O/st${n}_auto.err
done
timeout 900 python -m pytest tests/test_gpu_c5.py -q -x 2>&1 | tail -3 > $O/pytest.txt
