# Round-2 evaluation pass on one B200 (gpurun): newsvendor parity + sanitizers, the full
# bench line, the C2 epoch launch list and ncu --set full captures of its kernels.
set -u
mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_gpu_newsvendor.py tests/test_gpu_sharded.py -x -q > gpurun_out/r02/nvtests.log 2>&1; echo "rc $?" >> gpurun_out/r02/nvtests.log
if [ "${SAN:-0}" = 1 ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_paths.py nv > gpurun_out/r02/san_${tool}_nv.log 2>&1; echo "rc $?" >> gpurun_out/r02/san_${tool}_nv.log
  done
  SIMOPT_NV_QCAP=1 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_paths.py nv > gpurun_out/r02/san_memcheck_nv_qcap1.log 2>&1; echo "rc $?" >> gpurun_out/r02/san_memcheck_nv_qcap1.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err; echo "rc $?" >> gpurun_out/r02/bench.err
if [ "${NCU:-1}" = 1 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02/launches_nv_epoch.csv python tools/profile_nv.py > /dev/null 2>&1
  for k in k_nv_resample_ws k_nv_iter k_nv_records; do
    ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/r02/full_$k python tools/profile_nv.py > gpurun_out/r02/ncu_$k.log 2>&1
  done
fi
