R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
MD_AR_LL_MAX=1048576 timeout 600 $R --nproc-per-node 2 --master-port 29691 bench_sweep.py --max-mb 1 --no-eager --no-nccl --out gpurun_out/msw2.csv > gpurun_out/msw2.log 2>&1
MD_AR_LL_MAX=1048576 timeout 600 $R --nproc-per-node 4 --master-port 29692 bench_sweep.py --max-mb 1 --no-eager --no-nccl --out gpurun_out/msw4.csv > gpurun_out/msw4.log 2>&1
