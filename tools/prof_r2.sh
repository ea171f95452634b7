# Round-2 profile set (GPU box): bench line, launch list, ncu --set full of every
# tensor-core kernel for B_d1, C_d1, C_d8, D_d2 and E (fwd + bwd, 2nd iteration).
# The .ncu-rep files are summarised ON the box (tools/ncu_summary.py, raw CSV
# pages kept) and then moved out of gpurun_out/, which must stay < 64 MiB.
# usage: bash tools/prof_r2.sh TAG [configs...]
V=${1:-r2}
shift
CFGS=${@:-B_d1 C_d1 C_d8 D_d2 E}
mkdir -p /tmp/ncurep
python bench.py > gpurun_out/bench_$V.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fna_ -c 200 --csv --log-file gpurun_out/launches_$V.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_$V.csv gpurun_out/launches_$V.md
for C in $CFGS; do
  n=3; case $C in B_*) n=3;; *) n=4;; esac
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:fna_ -s $n -c $n -o /tmp/ncurep/full_${C}_$V python tools/run_fwd.py $C bwd > gpurun_out/ncu_${C}_$V.log 2>&1
  python tools/ncu_summary.py full /tmp/ncurep/full_${C}_$V.ncu-rep gpurun_out/ncu_full_${C}_$V.md gpurun_out/traffic_${C}_$V.json >> gpurun_out/ncu_${C}_$V.log 2>&1
  ncu -i /tmp/ncurep/full_${C}_$V.ncu-rep --page raw --csv > gpurun_out/raw_${C}_$V.csv 2>/dev/null
done
du -sh gpurun_out
