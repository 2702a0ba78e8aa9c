# round-2 quick check on a 2-GPU box: new routes/tests, bench N=1/2 (both update modes), stress
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out/q
python tools/nvlink_probe.py > gpurun_out/q/nvlink_probe.json 2>&1
timeout 900 python -m pytest tests/test_gpu_c5.py tests/test_gpu_stream.py -q -x 2>&1 | tail -15 > gpurun_out/q/pytest_c5.txt
timeout 900 python -m pytest tests/test_gpu_allreduce.py tests/test_gpu_owner.py -q -x 2>&1 | tail -15 > gpurun_out/q/pytest_ar.txt
timeout 300 python bench.py > gpurun_out/q/b1.json 2> gpurun_out/q/b1.err
timeout 300 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/q/b2.json 2> gpurun_out/q/b2.err
timeout 300 $R --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 --update sharded --no-cpu-baseline > gpurun_out/q/b2s.json 2> gpurun_out/q/b2s.err
timeout 400 $R --nproc-per-node 2 --master-port 29603 tools/stress_fused.py --calls 500 > gpurun_out/q/st2.json 2> gpurun_out/q/st2.err
timeout 400 $R --nproc-per-node 2 --master-port 29604 tools/stress_fused.py --calls 500 --sharded > gpurun_out/q/st2s.json 2> gpurun_out/q/st2s.err
