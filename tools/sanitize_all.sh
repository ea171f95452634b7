for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $t --error-exitcode 17 python tools/run_small.py > gpurun_out/san_$t.log 2>&1
  echo "rc=$?"; tail -3 gpurun_out/san_$t.log
done
