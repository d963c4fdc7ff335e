# compute-sanitizer pass over the round-2 session-3 changes: the serving loop's
# admission windows (shared-memory finish histograms and atomics, warp scans,
# the per-CTA decode-product table, per-lane product columns) and the sim_eval
# clock scan's jump-free fast path.  Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SAN="compute-sanitizer --print-limit 50 --error-exitcode 99 --target-processes all"
K1="sim_run_bit_exact or sim_eval or max_batch"
F="tests/test_gpu_fuzz.py::test_sim_run_window_edges"
K2="$F[0] $F[1] $F[2] $F[3] $F[7]"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $SAN --tool $tool python -m pytest tests/test_gpu_kernels.py -q -x -k "$K1" \
      -p no:cacheprovider > gpurun_out/san4_k_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/san4_k_${tool}.log
  timeout 1500 $SAN --tool $tool python -m pytest $K2 -q -x \
      -p no:cacheprovider > gpurun_out/san4_f_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/san4_f_${tool}.log
done
