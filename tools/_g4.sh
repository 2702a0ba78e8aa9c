R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $R --nproc-per-node 2 --master-port 29641 bench_sweep.py --max-mb 64 --out gpurun_out/sw2.csv > gpurun_out/sw2.log 2>&1
