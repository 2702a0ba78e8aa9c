R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
MD_AR_TRACE=1 timeout 300 $R --nproc-per-node 2 --master-port 29621 tools/trace_ar.py > gpurun_out/tr_n2.log 2>&1
mkdir -p gpurun_out/n2; mv gpurun_out/trace_n2_r*.bin gpurun_out/n2/
MD_AR_TRACE=1 timeout 300 $R --nproc-per-node 4 --master-port 29622 tools/trace_ar.py > gpurun_out/tr_n4.log 2>&1
mkdir -p gpurun_out/n4; mv gpurun_out/trace_n4_r*.bin gpurun_out/n4/
