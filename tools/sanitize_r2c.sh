# compute-sanitizer pass over the kernels added in the last round-2 session:
# the record grouping + list-mode SHA-256 + digest copy of dooly_dedup, the
# per-position / shared-memory-plane attention grid fit and the per-warp
# bulk-copy ring kernel (cp.async.bulk + mbarrier), and the sim_run in-order
# sums through shared memory.  Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SAN="compute-sanitizer --print-limit 50 --error-exitcode 99 --target-processes all"
K1="record_grouping or dedup_bit_exact or single_call or sim_run_bit_exact or sim_eval or iter_eval"
K2="ring or matches_oracle_and_csr"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $SAN --tool $tool python -m pytest tests/test_gpu_kernels.py -q -x -k "$K1" \
      -p no:cacheprovider > gpurun_out/san3_k_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/san3_k_${tool}.log
  timeout 1500 $SAN --tool $tool python -m pytest tests/test_gpu_fit_grid.py -q -x -k "$K2" \
      -p no:cacheprovider > gpurun_out/san3_g_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/san3_g_${tool}.log
done
