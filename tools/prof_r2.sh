# Round-2 profile set (GPU box): bench line, launch list, ncu --set full of every
# tensor-core kernel for B_d1, C_d1, C_d8, D_d2 and E (fwd + bwd, 2nd iteration).
# usage: bash tools/prof_r2.sh TAG
V=${1:-r2}
python bench.py > gpurun_out/bench_$V.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fna_ -c 200 --csv --log-file gpurun_out/launches_$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config > /dev/null 2>&1
for C in B_d1 C_d1 C_d8 D_d2 E; do
  n=3; case $C in B_*) n=3;; *) n=4;; esac
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:fna_ -s $n -c $n -o gpurun_out/full_${C}_$V python tools/run_fwd.py $C bwd > gpurun_out/ncu_${C}_$V.log 2>&1
done
ls gpurun_out
