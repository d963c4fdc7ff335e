# compute-sanitizer pass over the GPU tests of the atomics / bulk-copy rings /
# peer-store paths.  Run under gpurun from the repo root;
# logs go to gpurun_out/san_*.log, summaries into profiles/ by hand.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SAN="compute-sanitizer --print-limit 50 --error-exitcode 99 --target-processes all"
K="dedup or sha256 or record_hash or fit_matches or fit_exact or rank_deficient or predict_bit_exact or unknown or sim_run_bit_exact or sim_eval or iter_eval or non_termination"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $SAN --tool $tool python -m pytest tests/test_gpu_kernels.py -q -x -k "$K" \
      -p no:cacheprovider > gpurun_out/san_${tool}_kernels.log 2>&1
  echo "rc=$?" >> gpurun_out/san_${tool}_kernels.log
done
# shared-grid fit (cp.async.bulk / mbarrier rings), small sizes
for tool in memcheck racecheck synccheck; do
  timeout 900 $SAN --tool $tool python -m pytest tests/test_gpu_fit_grid.py -q -x \
      -p no:cacheprovider > gpurun_out/san_${tool}_fitgrid.log 2>&1
  echo "rc=$?" >> gpurun_out/san_${tool}_fitgrid.log
done
# routed dedup kernels + communicator (world 1 NCCL), and the fused peer-store
# path across two processes sharing the GPU (memcheck only)
timeout 900 $SAN --tool memcheck python -m pytest tests/test_gpu_comm.py -q -x \
    -p no:cacheprovider > gpurun_out/san_memcheck_comm.log 2>&1
echo "rc=$?" >> gpurun_out/san_memcheck_comm.log
timeout 1200 $SAN --tool memcheck python -m pytest tests/test_gpu_multirank.py -q -x -k "not bench" \
    -p no:cacheprovider > gpurun_out/san_memcheck_multirank.log 2>&1
echo "rc=$?" >> gpurun_out/san_memcheck_multirank.log
