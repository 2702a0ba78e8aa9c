# fused-step A/B at N=2: tree (default) vs the all-pull stream kernel at several tiles
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
port=29750
run() {  # label n env...
  label=$1; n=$2; shift 2
  port=$((port+1)); out=gpurun_out/st_${label}_n$n.json
  env "$@" timeout 300 $R --nproc-per-node $n --master-port $port bench.py --gpus $n --no-e2e > $out 2> $out.err
  python -c "import json; d=json.load(open('$out')); print('N=$n $label', round(d['step_ms']*1000,2), 'us/step', round(d['allreduce']['ms']*1000,2), 'us ar', round(d['roofline']['frac'],3))" || tail -5 $out.err
}
for rep in a b; do
  run tree$rep 2 MD_AR_STREAM=0
  for t in ${TILES:-5120 6144 6656 7168}; do run stream$t$rep 2 MD_AR_STREAM=1 MD_AR_TILE=$t; done
done
