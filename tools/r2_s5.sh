R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s5; mkdir -p $O
# ncu on one rank: where does it stop?
MASTER_PORT=29721 bash tools/ncu_rank0.sh 2 $O/ncu_diag.csv allreduce tools/ncu_diag.py > $O/ncu_diag.log 2>&1
# DIMD at N=4, push vs pull
for x in push pull; do
  timeout 600 $R --nproc-per-node 4 --master-port 29607 bench_dimd.py --exchange $x > $O/d4_$x.json 2> $O/d4_$x.err
done
# sharded tile sweep
for t in 0 1024 1536 2048 2560 3584 4096; do
  MD_AR_TILE=$t timeout 200 $R --nproc-per-node 2 --master-port 29608 tools/ar_call.py --update sharded --calls 12 > $O/tile2_$t.json 2>&1
done
for t in 0 1024 1536 2560 3072; do
  MD_AR_TILE=$t timeout 200 $R --nproc-per-node 4 --master-port 29609 tools/ar_call.py --update sharded --calls 12 > $O/tile4_$t.json 2>&1
done
# C2 sweeps
timeout 900 $R --nproc-per-node 2 --master-port 29610 bench_sweep.py --out $O/sweep_n2.csv > $O/sweep2.log 2>&1
timeout 900 $R --nproc-per-node 4 --master-port 29611 bench_sweep.py --out $O/sweep_n4.csv > $O/sweep4.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > $O/pytest.txt
