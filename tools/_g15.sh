R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_owner.py -q -x 2>&1 | tail -15 > gpurun_out/W_pytest.txt
timeout 900 $R --nproc-per-node 4 --master-port 29605 bench_sweep.py --no-eager --no-nccl --out gpurun_out/W_sweep_n4.csv > gpurun_out/W_sweep4.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 --no-e2e > gpurun_out/W_b4.json 2> gpurun_out/W_b4.err
