set -u
export PYTHONUNBUFFERED=1
for tool in memcheck synccheck racecheck; do
  for path in nv fused hessian; do
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_paths.py $path > gpurun_out/san_${tool}_${path}.log 2>&1
    echo "$tool $path rc=$?"
  done
done
for tool in memcheck synccheck; do
  port=$((29500 + RANDOM % 1000))
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_paths.py peer 0 2 $port > gpurun_out/san_${tool}_peer0.log 2>&1 &
  a=$!
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_paths.py peer 1 2 $port > gpurun_out/san_${tool}_peer1.log 2>&1
  b=$?
  wait $a; echo "$tool peer rc=$? $b"
done
