# A/B of environment knobs on one config: bench device value per setting, interleaved.
#   bash scripts/r02_env_ab_cfg.sh c5 "BE_X=1" "BE_X=0" ...
cfg=$1; shift
for v in "$@"; do
  env $v python bench.py --config $cfg --no-cpu --no-live --no-e2e --no-roofline --no-spec --steps 20 > gpurun_out/envab.json 2>gpurun_out/envab.err
  python -c "import json; d=json.loads(open('gpurun_out/envab.json').read().strip().splitlines()[-1]); print('$cfg $v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/envab.err
done
