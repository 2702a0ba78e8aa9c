R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s7; mkdir -p $O
for n in 2 4; do
  MD_AR_TRACE=1 timeout 200 $R --nproc-per-node $n --master-port 29641 tools/trace_push.py > $O/trace_n${n}_sharded.json 2> $O/trace_n${n}_sharded.err
  MD_AR_TRACE=1 timeout 200 $R --nproc-per-node $n --master-port 29642 tools/trace_push.py --update none > $O/trace_n${n}_plain.json 2> $O/trace_n${n}_plain.err
done
timeout 120 python tools/h2d_split_probe.py > $O/h2d_split.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
