# round-2 final pass (final code) on one 4-GPU box
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/final3; mkdir -p $O
nvidia-smi -L > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/pytest.txt
timeout 900 python -m pytest tests -m multigpu -v 2>&1 | grep -E "PASSED|FAILED|SKIPPED|ERROR|passed|failed" > $O/pytest_multigpu_list.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 400 python bench.py > $O/b1.json 2> $O/b1.err
timeout 400 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > $O/b2.json 2> $O/b2.err
timeout 400 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > $O/b4.json 2> $O/b4.err
timeout 400 python bench.py --impl reference > $O/r1.json 2> $O/r1.err
timeout 400 $R --nproc-per-node 2 --master-port 29603 bench.py --impl reference --gpus 2 > $O/r2.json 2> $O/r2.err
timeout 400 $R --nproc-per-node 4 --master-port 29604 bench.py --impl reference --gpus 4 > $O/r4.json 2> $O/r4.err
timeout 900 $R --nproc-per-node 2 --master-port 29610 bench_sweep.py --out $O/sweep_n2.csv > $O/sweep2.log 2>&1
timeout 900 $R --nproc-per-node 4 --master-port 29611 bench_sweep.py --out $O/sweep_n4.csv > $O/sweep4.log 2>&1
timeout 600 $R --nproc-per-node 1 --master-port 29605 bench_dimd.py > $O/d1.json 2> $O/d1.err
timeout 600 $R --nproc-per-node 2 --master-port 29606 bench_dimd.py > $O/d2.json 2> $O/d2.err
timeout 600 $R --nproc-per-node 4 --master-port 29607 bench_dimd.py > $O/d4.json 2> $O/d4.err
timeout 400 $R --nproc-per-node 4 --master-port 29608 tools/stress_fused.py --calls 2000 --sharded > $O/st4_sharded.json 2> $O/st4_sharded.err
MASTER_PORT=29734 bash tools/ncu_rank0.sh 4 $O/ncu_n4_sharded.csv allreduce tools/ar_call.py --update sharded > $O/ncu_n4_sharded.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi_end.txt
