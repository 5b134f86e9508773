#!/bin/bash
# Encoder iteration: GPU tests, path counts, bench (batched + per call), the
# launch list and one ncu --set full capture of one kernel launch.
#   tools/gpu_k2s.sh <tag> [kernel-regex] [launch-skip] [workload]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-k2s}; kre=${2:-^k_encode_small}; skip=${3:-2}; wl=${4:-hacc280m}
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 300 python tools/path_counts.py hacc280m > gpurun_out/${tag}_paths.txt 2>&1; timeout 300 python tools/path_counts.py lidar500m >> gpurun_out/${tag}_paths.txt 2>&1
timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu --per-call > gpurun_out/${tag}_bench_pc.json 2>> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --workload $wl --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 -o /tmp/${tag}_prof -f \
    python bench.py --workload $wl --steps 1 --warmup 1 --no-e2e --no-cpu --per-call --compress-only > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}_prof.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
ls -la gpurun_out | grep $tag
