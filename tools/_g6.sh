R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 120 $R --nproc-per-node 2 --master-port 29661 tools/oneshot_dbg.py > gpurun_out/dbg.log 2>&1
DBG_N=300000 timeout 120 $R --nproc-per-node 2 --master-port 29662 tools/oneshot_dbg.py > gpurun_out/dbg2.log 2>&1
