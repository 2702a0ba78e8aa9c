# round-2 session on a 4-GPU box: ncu pass diagnostics, NVLS probe, bench N=1/2/4 x update mode,
# stress at N=2/4, DIMD push vs pull, full GPU tests, smoke
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s4; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 120 ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum -c 2 ./tools/p2p_probe 64 > $O/ncu_pass_nvl.txt 2>&1
timeout 120 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum -c 2 ./tools/p2p_probe 64 > $O/ncu_pass_nvl_time.txt 2>&1
timeout 300 ./tools/nvls_probe 256 10 > $O/nvls_n4.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 300 ./tools/nvls_probe 256 10 > $O/nvls_n2.txt 2>&1
timeout 300 python bench.py > $O/b1.json 2> $O/b1.err
for u in replicated sharded; do
  timeout 300 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 --update $u --no-cpu-baseline > $O/b2_$u.json 2> $O/b2_$u.err
  timeout 300 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 --update $u --no-cpu-baseline > $O/b4_$u.json 2> $O/b4_$u.err
done
for n in 2 4; do
  timeout 400 $R --nproc-per-node $n --master-port 29603 tools/stress_fused.py --calls 2000 > $O/st${n}_auto.json 2> $O/st${n}_auto.err
  timeout 400 $R --nproc-per-node $n --master-port 29604 tools/stress_fused.py --calls 2000 --sharded > $O/st${n}_sharded.json 2> $O/st${n}_sharded.err
  timeout 400 $R --nproc-per-node $n --master-port 29605 tools/stress_fused.py --calls 2000 --route tree > $O/st${n}_tree.json 2> $O/st${n}_tree.err
  MD_AR_SYS_FENCE=1 timeout 400 $R --nproc-per-node $n --master-port 29606 tools/stress_fused.py --calls 2000 --route tree > $O/st${n}_tree_sys.json 2> $O/st${n}_tree_sys.err
done
for x in push pull; do
  timeout 600 $R --nproc-per-node 4 --master-port 29607 bench_dimd.py --exchange $x --cpu-records 0 > $O/d4_$x.json 2> $O/d4_$x.err
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $O/pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
