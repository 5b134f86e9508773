#!/bin/bash
# A/B of the in-tree library against every build/*.so, interleaved, R rounds
# (default 2) on the workloads in WLS (default hacc280m).
#   tools/gpu_ab_multi.sh <tag>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1
for wl in ${WLS:-hacc280m}; do
  for i in $(seq ${R:-2}); do
    for lib in paper_2508_10305_b200/_gpzb.so $(ls build/*.so); do
      echo "== $wl $i $lib" >> gpurun_out/${tag}_ab.txt
      GPZB_LIB=$PWD/$lib timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu $BENCH_ARGS 2>&1 \
        | python tools/ab_line.py >> gpurun_out/${tag}_ab.txt
    done
  done
done
cat gpurun_out/${tag}_ab.txt
