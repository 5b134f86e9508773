#!/bin/bash
# A/B of (library, environment) variants, interleaved, R rounds:
#   VARIANTS="base|paper_2508_10305_b200/_gpzb.so| cap1|build/cap.so|GPZB_K4W_CAP_P0=1" tools/gpu_ab_env.sh <tag>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1
for wl in ${WLS:-hacc280m}; do
  for i in $(seq ${R:-2}); do
    for v in $VARIANTS; do
      IFS='|' read -r name lib envs <<< "$v"
      echo "== $wl $i $name" >> gpurun_out/${tag}_ab.txt
      env $(echo $envs | tr ',' ' ') GPZB_LIB=$PWD/$lib timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu $BENCH_ARGS 2>&1 \
        | python tools/ab_line.py >> gpurun_out/${tag}_ab.txt
    done
  done
done
cat gpurun_out/${tag}_ab.txt
