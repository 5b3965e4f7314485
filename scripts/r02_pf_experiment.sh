for v in default pf4 pf8 pf16 default; do
  if [ $v = default ]; then L=""; else L="BE_LIB_PATH=scripts/variants/libblockexec_$v.so"; fi
  env $L python bench.py --no-cpu --no-live --no-e2e --no-roofline --steps 30 > gpurun_out/pf_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pf_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
for v in pf8 pf16; do BE_LIB_PATH=scripts/variants/libblockexec_$v.so python scripts/gemm_floor.py; done
