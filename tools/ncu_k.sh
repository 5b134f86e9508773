#!/bin/bash
# ncu --set full of K2 (pos + vel launches) and K4 with a given library (GPZB_LIB)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-cur}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_encode$" -s 2 -c 2 -o gpurun_out/prof_encode_$tag -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_encode_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_decode_warp$" -s 2 -c 2 -o gpurun_out/prof_decode_$tag -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_decode_$tag.log 2>&1
