# sanity.sh on a 4-GPU box: tests (multi-GPU thread paths included), smoke, bench N=1/2/4
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/S_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/S_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/S_smoke.txt 2>&1
timeout 300 python bench.py > gpurun_out/S_b1.json 2> gpurun_out/S_b1.err
timeout 300 $R --nproc-per-node 2 --master-port 29601 bench.py --gpus 2 > gpurun_out/S_b2.json 2> gpurun_out/S_b2.err
timeout 300 $R --nproc-per-node 4 --master-port 29602 bench.py --gpus 4 > gpurun_out/S_b4.json 2> gpurun_out/S_b4.err
