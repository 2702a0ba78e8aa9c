# Ready for an 8-GPU box (gpurun offers at most 4 here): the N = 8 rows of
# BASELINE configs C2-C5. C2: bench_sweep plans k = 1, 2, 4 (arity 4) and
# k = 8 (arity 7) at N = 8 and skips nothing else;
# C3/C5: bench.py (sharded fused update) and the replicated tree for
# comparison; C4: 8 x 160,000 records = the full 1.28M-record corpus; the
# cross-GPU protocol stress at N = 8.
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/n8; mkdir -p $O
timeout 1500 python -m pytest tests -m multigpu -q 2>&1 | tail -3 > $O/pytest_multigpu.txt
timeout 600 $R --nproc-per-node 8 --master-port 29601 bench.py --gpus 8 > $O/b8.json 2> $O/b8.err
timeout 600 $R --nproc-per-node 8 --master-port 29602 bench.py --gpus 8 --update replicated --no-cpu-baseline > $O/b8_repl.json 2> $O/b8_repl.err
timeout 600 $R --nproc-per-node 8 --master-port 29603 bench.py --impl reference --gpus 8 > $O/r8.json 2> $O/r8.err
timeout 1200 $R --nproc-per-node 8 --master-port 29604 bench_sweep.py --out $O/sweep_n8.csv > $O/sweep8.log 2>&1
timeout 900 $R --nproc-per-node 8 --master-port 29605 bench_dimd.py > $O/d8.json 2> $O/d8.err
timeout 600 $R --nproc-per-node 8 --master-port 29606 tools/stress_fused.py --calls 2000 --sharded > $O/st8_sharded.json 2> $O/st8_sharded.err
timeout 600 $R --nproc-per-node 8 --master-port 29607 tools/stress_fused.py --calls 2000 > $O/st8_auto.json 2> $O/st8_auto.err
