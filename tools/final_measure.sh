# Consolidated round measurement on one 4-GPU box (gpurun --gpus 4):
#   GPU tests, bench N=1/2/4 (+ reference arm), C2 sweeps N=2/4, DIMD C4 N=1/2/4,
#   ncu launch list + full capture of the fused kernel (N=1, single process).
set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/F_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/F_smoke.txt 2>&1
python bench.py > gpurun_out/F_b1.json 2> gpurun_out/F_b1.err
$R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > gpurun_out/F_b2.json 2> gpurun_out/F_b2.err
$R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > gpurun_out/F_b4.json 2> gpurun_out/F_b4.err
python bench.py --impl reference > gpurun_out/F_r1.json 2> gpurun_out/F_r1.err
$R --nproc-per-node 2 --master-port 29603 bench.py --impl reference --gpus 2 > gpurun_out/F_r2.json 2> gpurun_out/F_r2.err
$R --nproc-per-node 4 --master-port 29604 bench.py --impl reference --gpus 4 > gpurun_out/F_r4.json 2> gpurun_out/F_r4.err
$R --nproc-per-node 2 --master-port 29605 bench_sweep.py --out gpurun_out/F_sweep_n2.csv > gpurun_out/F_sweep2.log 2>&1
$R --nproc-per-node 4 --master-port 29606 bench_sweep.py --out gpurun_out/F_sweep_n4.csv > gpurun_out/F_sweep4.log 2>&1
$R --nproc-per-node 1 --master-port 29607 bench_dimd.py > gpurun_out/F_d1.json 2> gpurun_out/F_d1.err
$R --nproc-per-node 2 --master-port 29608 bench_dimd.py > gpurun_out/F_d2.json 2> gpurun_out/F_d2.err
$R --nproc-per-node 4 --master-port 29609 bench_dimd.py > gpurun_out/F_d4.json 2> gpurun_out/F_d4.err
MD_BENCH_NOCLOCK=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/F_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/F_ncu1.log 2>&1
MD_BENCH_NOCLOCK=1 ncu --set full --clock-control none --import-source on -k regex:sgd_vec_kernel \
  -s 3 -c 1 -o gpurun_out/F_ar_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/F_ncu2.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/F_smi.txt
