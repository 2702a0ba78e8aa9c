# segment-size sweep of the fused allreduce at N=2 and N=4 (tools/diag_ar.py)
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
export DIAG_NOSYNC=1 DIAG_NOSTEP=1 DIAG_SEGS=${DIAG_SEGS:-2048,4096,8192,16384,32768}
timeout 300 $R --nproc-per-node 2 --master-port 29611 tools/diag_ar.py > gpurun_out/seg_n2.log 2>&1
timeout 300 $R --nproc-per-node 4 --master-port 29612 tools/diag_ar.py > gpurun_out/seg_n4.log 2>&1
