# Kernel-variant sweep of the shared-grid fit at C5 size (tools/fit_grid_bench.py).
python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 > gpurun_out/fg_default.jsonl
DOOLY_FIT_GRID_KERNEL=warp python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 > gpurun_out/fg_warp.jsonl
for ys in 2 4; do
DOOLY_FIT_GRID_KERNEL=pair DOOLY_FIT_GRID_YS=$ys python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 --vs-warp > gpurun_out/fg_pair_${ys}.jsonl 2>&1
done
