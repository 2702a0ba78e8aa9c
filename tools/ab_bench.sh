# A/B of bench.py under an env switch: tools/ab_bench.sh VAR [Ns...]
# prints one summary line per (N, setting); full JSON under gpurun_out/ab_*
VAR=$1; shift
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29700
for n in "$@"; do
  for set in 0 1; do
    port=$((port+1))
    if [ $set = 1 ]; then export $VAR=1; else unset $VAR; fi
    out=gpurun_out/ab_${VAR}_${set}_n$n.json
    if [ $n = 1 ]; then
      timeout 300 python bench.py --no-cpu-baseline --no-e2e > $out 2> $out.err
    else
      timeout 300 $R --nproc-per-node $n --master-port $port bench.py --gpus $n --no-e2e > $out 2> $out.err
    fi
    python -c "import json,sys; d=json.load(open('$out')); print('N=$n $VAR=$set', round(d['step_ms']*1000,2), 'us/step', round(d['allreduce']['ms']*1000,2), 'us ar', d['roofline']['frac'])" || tail -5 $out.err
  done
done
unset $VAR
