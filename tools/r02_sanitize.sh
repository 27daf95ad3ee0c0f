# compute-sanitizer over the round-2 kernels (newsvendor step/records, fused async exchange,
# persistent mean-variance epoch); logs in gpurun_out/r02san/
set -u
mkdir -p gpurun_out/r02san
for tool in memcheck racecheck synccheck; do
  for path in nv fused; do
    timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_paths.py $path > gpurun_out/r02san/${tool}_${path}.log 2>&1; echo "rc $?" >> gpurun_out/r02san/${tool}_${path}.log
  done
done
