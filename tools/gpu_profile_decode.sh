#!/bin/bash
# ncu full captures of K4w (pos + vel launches) and K3b.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_decode_warp$" -s 2 -c 2 -o gpurun_out/prof_decode -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_decode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_copy_payloads$" -s 2 -c 1 -o gpurun_out/prof_copy -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_copy.log 2>&1
