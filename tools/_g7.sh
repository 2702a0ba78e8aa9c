R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $R --nproc-per-node 2 --master-port 29671 bench_sweep.py --max-mb 1 --no-eager --no-nccl --out gpurun_out/x1.csv > gpurun_out/x1.log 2>&1
timeout 300 $R --nproc-per-node 2 --master-port 29672 bench_sweep.py --max-mb 1 --no-eager --out gpurun_out/x2.csv > gpurun_out/x2.log 2>&1
