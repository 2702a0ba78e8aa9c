# work-queue tree kernel at 384 threads (no spills): parity + stress + timing at N=2
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s16; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_allreduce.py tests/test_gpu_c5.py -m gpu -q 2>&1 | tail -5 > $O/pytest.txt
timeout 600 $R --nproc-per-node 2 --master-port 29630 tools/stress_fused.py --calls 1000 --route queue > $O/stress_queue.json 2> $O/stress_queue.err
timeout 300 $R --nproc-per-node 2 --master-port 29631 tools/ar_call.py --route queue --update replicated > $O/ar_queue.json 2> $O/ar_queue.err
timeout 300 $R --nproc-per-node 2 --master-port 29632 tools/ar_call.py --route tree --update replicated > $O/ar_tree.json 2> $O/ar_tree.err
