# Round-2 final multi-GPU runs on a 4-GPU box: block placement bench lines (C2, C4, C5 with its
# speculation leg) at 2 and 4 GPUs, NCCL-vs-loopback bit-exactness at 2 and 4.
mkdir -p gpurun_out/final
for N in 2 4; do
  for c in c2 c4 c5; do
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 2960$N bench.py --gpus $N --config $c --steps 20 --warmup 5 \
      > gpurun_out/final/bench_n${N}_$c.json 2> gpurun_out/final/bench_n${N}_$c.err
    python -c "import json; d=json.loads(open('gpurun_out/final/bench_n${N}_$c.json').read().strip().splitlines()[-1]); r=d.get('replicas') or {}; s=d.get('speculation') or {}; print('$N $c', d['value'], r.get('value'), (d.get('e2e') or {}).get('value'), s.get('tokens_per_s'), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/final/bench_n${N}_$c.err
  done
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2970$N scripts/cluster_check.py --config c2 > gpurun_out/final/cc_n$N.log 2>&1; tail -c 400 gpurun_out/final/cc_n$N.log
done
