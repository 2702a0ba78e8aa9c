R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/S_pytest.txt
timeout 300 $R --nproc-per-node 2 --master-port 29701 bench.py --gpus 2 --no-e2e > gpurun_out/S_b2.json 2> gpurun_out/S_b2.err
MD_AR_STREAM=0 timeout 300 $R --nproc-per-node 2 --master-port 29702 bench.py --gpus 2 --no-e2e > gpurun_out/S_b2t.json 2> gpurun_out/S_b2t.err
timeout 600 $R --nproc-per-node 2 --master-port 29703 bench_sweep.py --no-eager --no-nccl --out gpurun_out/ssw2.csv > gpurun_out/ssw2.log 2>&1
MD_AR_ONESHOT_MAX=0 timeout 600 $R --nproc-per-node 2 --master-port 29704 bench_sweep.py --max-mb 16 --no-eager --no-nccl --out gpurun_out/ssw2b.csv > gpurun_out/ssw2b.log 2>&1
