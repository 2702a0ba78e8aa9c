R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python bench.py > gpurun_out/Z_b1.json 2> gpurun_out/Z_b1.err
timeout 300 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > gpurun_out/Z_b2.json 2> gpurun_out/Z_b2.err
timeout 300 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > gpurun_out/Z_b4.json 2> gpurun_out/Z_b4.err
