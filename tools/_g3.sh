R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python bench.py > gpurun_out/Q_b1.json 2> gpurun_out/Q_b1.err
timeout 300 $R --nproc-per-node 2 --master-port 29631 bench.py --gpus 2 > gpurun_out/Q_b2.json 2> gpurun_out/Q_b2.err
timeout 300 $R --nproc-per-node 4 --master-port 29632 bench.py --gpus 4 > gpurun_out/Q_b4.json 2> gpurun_out/Q_b4.err
for n in 1 2 4; do python -c "import json; d=json.load(open('gpurun_out/Q_b$n.json')); print($n, round(d['step_ms']*1000,2), round(d['allreduce']['ms']*1000,2), d['roofline']['frac'], d['e2e']['value'], d['value'])"; done
