R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/G_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/G_smoke.txt 2>&1
timeout 300 python bench.py > gpurun_out/G_b1.json 2> gpurun_out/G_b1.err
timeout 300 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > gpurun_out/G_b2.json 2> gpurun_out/G_b2.err
timeout 300 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > gpurun_out/G_b4.json 2> gpurun_out/G_b4.err
timeout 900 $R --nproc-per-node 4 --master-port 29606 bench_sweep.py --no-eager --out gpurun_out/G_sweep_n4.csv > gpurun_out/G_sweep4.log 2>&1
timeout 900 $R --nproc-per-node 2 --master-port 29605 bench_sweep.py --no-eager --out gpurun_out/G_sweep_n2.csv > gpurun_out/G_sweep2.log 2>&1
