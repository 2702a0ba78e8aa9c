# round-2 closing pass (one 4-GPU box): all GPU tests incl. multi-GPU, smoke,
# C5 bench N=1/2/4 + reference arm, C4 DIMD N=1/2/4
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/final5; mkdir -p $O
nvidia-smi -L > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/pytest.txt
timeout 900 python -m pytest tests -m multigpu -v 2>&1 | grep -E "PASSED|FAILED|SKIPPED|ERROR|passed|failed" > $O/pytest_multigpu_list.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 400 python bench.py > $O/b1.json 2> $O/b1.err
timeout 400 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > $O/b2.json 2> $O/b2.err
timeout 400 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > $O/b4.json 2> $O/b4.err
timeout 400 python bench.py --impl reference > $O/r1.json 2> $O/r1.err
timeout 600 $R --nproc-per-node 1 --master-port 29605 bench_dimd.py > $O/d1.json 2> $O/d1.err
timeout 600 $R --nproc-per-node 2 --master-port 29606 bench_dimd.py > $O/d2.json 2> $O/d2.err
timeout 600 $R --nproc-per-node 4 --master-port 29607 bench_dimd.py > $O/d4.json 2> $O/d4.err
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi_end.txt
