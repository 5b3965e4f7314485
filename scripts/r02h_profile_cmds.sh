set -x
python scripts/profile_step.py --out gpurun_out/r02h_step_prof.json > gpurun_out/r02h_ps.log 2>&1 &&
python scripts/profile_step.py --steps 1 > gpurun_out/plain.log 2>&1 &&
ncu --nvtx --nvtx-include step/ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02h_step_launches.csv python scripts/profile_step.py --steps 1 > gpurun_out/ncu1.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu --profile --no-e2e --no-live > gpurun_out/plain2.log 2>&1 &&
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02h_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --profile --no-e2e --no-live > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out/
