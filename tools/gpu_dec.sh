#!/bin/bash
# Decoder iteration: decode tests, bench, and one ncu --set full capture of
# the velocity K4w launch.   tools/gpu_dec.sh <tag> [kernel-regex] [skip]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-dec}; kre=${2:-^k_decode_warp}; skip=${3:-1}
timeout 900 python -m pytest tests -x -q -m gpu -k "decode or decompress or golden or bitflip or streamed or iter or warp" > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 -o /tmp/${tag}_prof -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --per-call > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}_prof.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
ls -la gpurun_out | grep $tag
