# Round-end evidence refresh on one B200 (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/rr_bench.json 2> gpurun_out/rr_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/rr_ref.json 2> gpurun_out/rr_ref.err
# the launch list of the default bench command (our kernels only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:'predict_|fit_|sha256|dedup_|sim_|iter_eval|attn_pack|profile_fit|peer_|route_|rec_group|digest_copy' \
    --log-file gpurun_out/rr_launches.csv python bench.py --steps 2 --warmup 1 \
    > gpurun_out/rr_launches_bench.log 2>&1
# full capture of the dominant kernel (the paired packed-attention predict)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:predict_attn_pair -c 1 \
    -o gpurun_out/rr_pair -f python tools/predict_sweep.py --sigs 500000 --queries 100000000 \
    --layouts attn96 --reps 1 > gpurun_out/rr_pair.log 2>&1
# full capture of the attention grid fit (grouped passes)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fit_grid_warp -c 1 \
    -o gpurun_out/rr_fgw -f python tools/fit_grid_bench.py --sigs 200000 --kinds 1 --reps 1 \
    > gpurun_out/rr_fgw.log 2>&1
# the driver's smoke entry point
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rr_smoke.log 2>&1
