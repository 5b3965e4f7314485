# A/B of environment knobs on one box: bench value (device step) per setting, interleaved.
#   bash scripts/r02_env_ab.sh "BE_ATTN_PF=1" "BE_ATTN_PF=0" ...
for v in "$@"; do
  env $v python bench.py --no-cpu --no-live --no-e2e --no-roofline --steps 30 > gpurun_out/envab.json 2>gpurun_out/envab.err
  python -c "import json; d=json.loads(open('gpurun_out/envab.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/envab.err
done
