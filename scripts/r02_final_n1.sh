# Round-2 final single-GPU validation: full GPU test suite, smoke, every config's bench line,
# the reference arm. Outputs under gpurun_out/final/.
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/final/pytest_gpu.log 2>&1; tail -3 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/final/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d.get('prefill_s'))" || tail -3 gpurun_out/final/bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; tail -c 300 gpurun_out/final/bench_reference.json
