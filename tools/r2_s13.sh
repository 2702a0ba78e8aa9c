R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s13; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dimd.py tests/test_gpu_multiproc.py tests/test_gpu_sgd.py -q -x 2>&1 | tail -5 > $O/pytest.txt
MD_DIMD_TIMING=1 timeout 600 $R --nproc-per-node 4 --master-port 29607 bench_dimd.py --cpu-records 0 --epochs 6 > $O/d4_timing.json 2> $O/d4_timing.err
timeout 600 $R --nproc-per-node 4 --master-port 29608 bench_dimd.py --epochs 6 --cpu-records 0 > $O/d4.json 2> $O/d4.err
timeout 600 $R --nproc-per-node 4 --master-port 29609 bench_dimd.py --epochs 6 --cpu-records 0 --no-prefetch-plan > $O/d4_noprefetch.json 2> $O/d4_noprefetch.err
timeout 600 $R --nproc-per-node 2 --master-port 29610 bench_dimd.py --epochs 6 --cpu-records 0 > $O/d2.json 2> $O/d2.err
