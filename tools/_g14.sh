export MD_BENCH_NOCLOCK=1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/N_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/N_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:allreduce_channels_kernel -s 3 -c 1 -o gpurun_out/N_ar_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/N_ncu2.log 2>&1
ncu -i gpurun_out/N_ar_full.ncu-rep --page raw --csv > gpurun_out/N_ar_full_raw.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q 2>&1 | tail -5 > gpurun_out/N_mp.txt
