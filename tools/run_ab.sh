# A/B of library builds (GPU box): bitwise check against the first, then
# per-kernel times of B_d1, C_d1, C_d8, D_d2, E for each, twice.
# usage: bash tools/run_ab.sh TAG base.so variant.so ...
TAG=$1; shift
python tools/ab_check.py "$@" > gpurun_out/ab_check_$TAG.log 2>&1
for L in "$@"; do
  python tools/time_variant.py $L B_d1 C_d1 C_d8 D_d2 E >> gpurun_out/ab_time_$TAG.log 2>&1
done
for L in "$@"; do
  python tools/time_variant.py $L B_d1 C_d1 C_d8 D_d2 E >> gpurun_out/ab_time_$TAG.log 2>&1
done
