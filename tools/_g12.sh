R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
export DIAG_NOSYNC=1 DIAG_NOSTEP=1 DIAG_SEGS=16384 MD_AR_STREAM=1
for te in 1024 2048 4096; do
MD_AR_TILE=$te timeout 300 $R --nproc-per-node 2 --master-port 2971${te:0:1} tools/diag_ar.py > gpurun_out/te_$te.log 2>&1
done
MD_AR_STREAM=0 timeout 300 $R --nproc-per-node 2 --master-port 29719 tools/diag_ar.py > gpurun_out/te_tree.log 2>&1
