for a in 1 2 3 4; do for t in 1 2; do
 DOOLY_FIT_STAGES_AFFINE=$a DOOLY_FIT_STAGES_ATTN=$t timeout 300 python bench.py --steps 3 --warmup 3 --queries 8000000 --sigs 200000 --records 0 --sim-requests 0 --e2e-queries 0 --cpu-sample 0 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('aff_st=$a attn_st=$t', d['fits']['kernel_ms'])"
done; done
