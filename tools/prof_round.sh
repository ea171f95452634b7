# Profile round: bench line, launch list, ncu --set full captures (B_d1, E backward+forward).
# usage (GPU box): bash tools/prof_round.sh TAG
V=${1:-v7}
set -x
python bench.py > gpurun_out/bench_$V.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fna_ -c 200 --csv --log-file gpurun_out/launches_$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fna_ -s 3 -c 3 -o gpurun_out/full_$V python tools/run_fwd.py B_d1 bwd > gpurun_out/ncu_full_$V.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fna_ -s 4 -c 4 -o gpurun_out/full_E_$V python tools/run_fwd.py E bwd > gpurun_out/ncu_full_E_$V.log 2>&1
tail -1 gpurun_out/bench_$V.log | cut -c1-300
ls -la gpurun_out
