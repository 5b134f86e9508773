#!/bin/bash
# Encoder routing experiment: per-call bench under each GPZB_ROUTE, launch list
# for the offset-free route, ncu of the position encoder.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-route}
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --per-call --compress-only > gpurun_out/${tag}_default.json 2>&1
GPZB_ROUTE=small0 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --per-call --compress-only > gpurun_out/${tag}_small0.json 2>&1
GPZB_ROUTE=small0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_small0_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --compress-only > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_encode_warp" -s 0 -c 1 -o /tmp/${tag}_prof -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --per-call --compress-only > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}_prof.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
ls -la gpurun_out | grep $tag
