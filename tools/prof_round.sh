set -x
python bench.py > gpurun_out/bench_v6.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fna_ -c 200 --csv --log-file gpurun_out/launches_v6.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fna_ -s 4 -c 4 -o gpurun_out/full_v6 python tools/run_fwd.py B_d1 bwd > gpurun_out/ncu_full_v6.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fna_ -s 4 -c 4 -o gpurun_out/full_E_v6 python tools/run_fwd.py E bwd > gpurun_out/ncu_full_E_v6.log 2>&1
tail -1 gpurun_out/bench_v6.log | cut -c1-300
ls -la gpurun_out
