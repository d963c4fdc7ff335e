# Round-end evidence refresh on one B200 (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/rr_bench.json 2> gpurun_out/rr_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/rr_ref.json 2> gpurun_out/rr_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'predict_vec|predict_scalar|fit_|sha256|dedup_|sim_run|iter_eval|attn_pack|profile_fit|peer_' \
    --log-file gpurun_out/rr_launches.csv python bench.py --steps 2 --warmup 1 \
    > gpurun_out/rr_launches_bench.log 2>&1
# full captures: the attention grid fit (grouped passes) and the CSR moments kernel
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fit_grid_warp -c 1 \
    -o gpurun_out/rr_fgw -f python tools/fit_grid_bench.py --sigs 200000 --kinds 1 --reps 1 \
    > gpurun_out/rr_fgw.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fit_moments_attn -c 1 \
    -o gpurun_out/rr_mom -f python tools/fit_grid_bench.py --sigs 60000 --kinds 1 --reps 1 --csr \
    > gpurun_out/rr_mom.log 2>&1
