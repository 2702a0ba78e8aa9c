R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/F_pytest.txt
timeout 300 python bench.py > gpurun_out/F_b1.json 2> gpurun_out/F_b1.err
timeout 300 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > gpurun_out/F_b2.json 2> gpurun_out/F_b2.err
timeout 300 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > gpurun_out/F_b4.json 2> gpurun_out/F_b4.err
timeout 900 $R --nproc-per-node 2 --master-port 29604 bench_sweep.py --out gpurun_out/F_sweep_n2.csv > gpurun_out/F_sweep2.log 2>&1
timeout 900 $R --nproc-per-node 4 --master-port 29605 bench_sweep.py --out gpurun_out/F_sweep_n4.csv > gpurun_out/F_sweep4.log 2>&1
