nvidia-smi topo -m > gpurun_out/H_topo.txt 2>&1
for i in 1 2; do timeout 300 python bench.py > gpurun_out/H_b1_$i.json 2> gpurun_out/H_b1_$i.err; done
timeout 300 python bench.py --impl reference > gpurun_out/H_r1.json 2> gpurun_out/H_r1.err
python tools/h2d_probe.py > gpurun_out/H_h2d.txt 2>&1
