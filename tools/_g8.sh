R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/L_pytest.txt
timeout 600 $R --nproc-per-node 2 --master-port 29681 bench_sweep.py --max-mb 64 --no-eager --out gpurun_out/lsw2.csv > gpurun_out/lsw2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29682 bench_sweep.py --max-mb 64 --no-eager --out gpurun_out/lsw4.csv > gpurun_out/lsw4.log 2>&1
MD_AR_ONESHOT_MAX=67108864 timeout 600 $R --nproc-per-node 4 --master-port 29683 bench_sweep.py --max-mb 64 --no-eager --no-nccl --out gpurun_out/lsw4b.csv > gpurun_out/lsw4b.log 2>&1
