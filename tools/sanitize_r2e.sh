# compute-sanitizer pass over the session-3 CSR fit kernels: the default
# warp-per-signature affine kernel and the opt-in fused attention kernel.
# Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SAN="compute-sanitizer --print-limit 50 --error-exitcode 99 --target-processes all"
T="tests/test_gpu_fuzz.py::test_fit_csr_affine_warp_large_ragged tests/test_gpu_fuzz.py::test_fit_csr_attn_fused_matches_split"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $SAN --tool $tool python -m pytest $T -q -x -p no:cacheprovider \
      > gpurun_out/san5_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/san5_${tool}.log
done
