# compute-sanitizer pass over the kernels changed late in round 2: the hybrid
# TMA gather4 + paired predict kernel (mbarrier ring), every packed-attention
# variant, the SHA-256 records kernel (stream state in registers) and both
# dedup insert kernels.  Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
SAN="compute-sanitizer --print-limit 50 --error-exitcode 99 --target-processes all"
K="cooperative_kernel or dedup_bit_exact or sha256 or record_hash or census"
for tool in memcheck racecheck synccheck; do
  timeout 1500 $SAN --tool $tool python -m pytest tests/test_gpu_kernels.py -q -x -k "$K" \
      -p no:cacheprovider > gpurun_out/san2_${tool}.log 2>&1
  echo "rc=$?" >> gpurun_out/san2_${tool}.log
done
