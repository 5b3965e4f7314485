# A/B of library variants on the end-to-end leg: bench e2e value per variant, interleaved
for v in "$@"; do
  L="BE_LIB_PATH=scripts/variants/libblockexec_$v.so"
  env $L python bench.py --no-cpu --no-live --no-roofline --steps 30 > gpurun_out/e2e_$v.json 2>gpurun_out/e2e_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/e2e_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], round(d['e2e']['value'],1), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/e2e_$v.err
done
