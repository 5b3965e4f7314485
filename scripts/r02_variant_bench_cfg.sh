# A/B of library variants on one config: bench device value per variant, interleaved.
#   bash scripts/r02_variant_bench_cfg.sh c5 staged chunked ...
cfg=$1; shift
for v in "$@"; do
  BE_LIB_PATH=scripts/variants/libblockexec_$v.so python bench.py --config $cfg --no-cpu --no-live --no-e2e --no-roofline --no-spec --steps 20 > gpurun_out/var_$v.json 2>gpurun_out/var_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1]); print('$cfg $v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/var_$v.err
done
