# Kernel-variant sweep of the shared-grid fit at C5 size (tools/fit_grid_bench.py).
python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 > gpurun_out/fg_default.jsonl
DOOLY_FIT_GRID_KERNEL=db DOOLY_FIT_GRID_YS=8 python tools/fit_grid_bench.py --sigs 500000 --kinds 0,1 --vs-warp > gpurun_out/fg_db8.jsonl 2>&1
DOOLY_FIT_GRID_KERNEL=warp DOOLY_FIT_GRID_WARPS=24 python tools/fit_grid_bench.py --sigs 500000 --kinds 1 > gpurun_out/fg_w24.jsonl 2>&1
