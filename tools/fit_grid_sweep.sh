# Kernel-variant sweep of the shared-grid fit at C5 size (tools/fit_grid_bench.py).
python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 > gpurun_out/fg_default.jsonl 2>&1
DOOLY_FIT_GRID_KERNEL=db python tools/fit_grid_bench.py --sigs 500000 --kinds 1 --vs-warp > gpurun_out/fg_db_grouped.jsonl 2>&1
