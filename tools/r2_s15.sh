# h2d placement probe: concurrent pinned H2D on every rank, default vs GPU-local NUMA node
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
O=gpurun_out/s15; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
cat /sys/devices/system/node/online > $O/nodes.txt 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29620 tools/h2d_numa_probe.py > $O/n4.json 2> $O/n4.err
timeout 300 $R --nproc-per-node 2 --master-port 29621 tools/h2d_numa_probe.py > $O/n2.json 2> $O/n2.err
timeout 300 $R --nproc-per-node 1 --master-port 29622 tools/h2d_numa_probe.py > $O/n1.json 2> $O/n1.err
