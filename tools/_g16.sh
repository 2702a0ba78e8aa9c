R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for sg in 2048 4096 8192; do
timeout 600 $R --nproc-per-node 4 --master-port 2961${sg:0:1} bench_sweep.py --max-mb 64 --seg $sg --no-eager --no-nccl --out gpurun_out/G_sw4_$sg.csv > gpurun_out/G_sw4_$sg.log 2>&1
timeout 600 $R --nproc-per-node 2 --master-port 2962${sg:0:1} bench_sweep.py --max-mb 64 --seg $sg --no-eager --no-nccl --out gpurun_out/G_sw2_$sg.csv > gpurun_out/G_sw2_$sg.log 2>&1
done
