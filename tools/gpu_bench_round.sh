#!/bin/bash
# One GPU round: full bench, ncu launch list, ncu full captures of K2 (pos+vel), K3b, K4 (pos+vel).
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_ncu.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_encode$" -s 1 -c 1 -o gpurun_out/prof_encode -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_encode.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_encode_warp$" -s 1 -c 1 -o gpurun_out/prof_encode_warp -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_encode_warp.log 2>&1
# (second call, the reports exceed gpurun's 64 MiB return limit together): tools/gpu_profile_decode.sh
ls -la gpurun_out
