# Kernel-variant sweep of the shared-grid fit at C5 size (tools/fit_grid_bench.py);
# run under gpurun from the repo root.  Lines land in gpurun_out/fg_*.jsonl.
#   defaults: db kernel (affine), warp kernel with grouped passes (attention)
python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 > gpurun_out/fg_default.jsonl 2>&1
# per-point attention passes, for the grouped-pass speed-up and coefficient agreement
python tools/fit_grid_bench.py --sigs 500000 --kinds 1 --vs-unfactored > gpurun_out/fg_grouped.jsonl 2>&1
# the other kernels, bit-identity against the warp kernel
for k in db stage; do
  DOOLY_FIT_GRID_KERNEL=$k python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 --vs-warp \
    > gpurun_out/fg_$k.jsonl 2>&1
done
# the per-signature CSR path on the same points
python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 --csr --reps 1 > gpurun_out/fg_csr.jsonl 2>&1
