R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/O_pytest.txt
timeout 600 $R --nproc-per-node 2 --master-port 29651 bench_sweep.py --max-mb 64 --no-eager --out gpurun_out/osw2.csv > gpurun_out/osw2.log 2>&1
timeout 600 $R --nproc-per-node 4 --master-port 29652 bench_sweep.py --max-mb 64 --no-eager --out gpurun_out/osw4.csv > gpurun_out/osw4.log 2>&1
