#!/bin/bash
# A/B of a library build on one box: the in-tree _gpzb.so vs build/<name>.so,
# alternating, batched bench (compress + decompress) twice each, plus the
# parity tests that exercise the encoders with the candidate.
#   tools/gpu_ab_lib.sh <tag> <name>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; cand=build/$2.so
GPZB_LIB=$cand timeout 900 python -m pytest tests -x -q -m gpu -k "golden or random or bench_workload or stress or velocity or configs or batched or large or bitflip or warp or streamed or iter" > gpurun_out/${tag}_pytest.txt 2>&1
echo "rc=$?" >> gpurun_out/${tag}_pytest.txt
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_base$i.json 2>&1
  GPZB_LIB=$cand timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_cand$i.json 2>&1
done
GPZB_LIB=$cand timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_cand_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --compress-only > /dev/null 2>&1
