# A/B of library variants on one box: bench value (device step) per variant, interleaved
for v in "$@"; do
  if [ $v = default ]; then L=""; else L="BE_LIB_PATH=scripts/variants/libblockexec_$v.so"; fi
  env $L python bench.py --no-cpu --no-live --no-e2e --no-roofline --steps 30 > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/var_$v.err
done
