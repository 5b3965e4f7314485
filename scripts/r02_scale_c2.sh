# C2 at 1, 2 and 4 GPUs back to back on one 4-GPU box (the driver's scaling run, block placement)
mkdir -p gpurun_out/final
python bench.py --steps 20 --warmup 5 --no-cpu --no-live > gpurun_out/final/scale_n1.json 2>/dev/null
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2980$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/final/scale_n$N.json 2>/dev/null
done
for N in 1 2 4; do
  python -c "import json; d=json.loads(open('gpurun_out/final/scale_n$N.json').read().strip().splitlines()[-1]); print($N, d['value'], d['e2e']['value'], d['clocks']['sm_mhz'], (d.get('replicas') or {}).get('value'))"
done
