#!/bin/bash
# A/B of encoder routes on one box: path counts and the batched bench under
# each GPZB_ROUTE value given.   tools/gpu_ab_route.sh <tag> route1 route2 ...
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; shift
for r in "$@"; do
  GPZB_ROUTE=$r timeout 300 python tools/path_counts.py hacc280m > gpurun_out/${tag}_${r}_paths.txt 2>&1
  for i in 1 2; do
    GPZB_ROUTE=$r timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --compress-only > gpurun_out/${tag}_${r}_bench$i.json 2>&1
  done
done
