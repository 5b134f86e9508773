#!/bin/bash
# A/B of build/<name>.so vs the in-tree library on hacc280m and lidar500m
# (alternating runs), after the encoder parity tests with the candidate
# (NOTEST=1 skips them).
#   tools/gpu_ab_wl.sh <tag> <name>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; cand=build/$2.so
if [ -z "$NOTEST" ]; then
  GPZB_LIB=$cand timeout 900 python -m pytest tests -x -q -m gpu -k "golden or random or bench_workload or stress or velocity or configs or batched or large or bitflip or streamed" > gpurun_out/${tag}_pytest.txt 2>&1
  echo "rc=$?" >> gpurun_out/${tag}_pytest.txt
  tail -3 gpurun_out/${tag}_pytest.txt
fi
for wl in ${WLS:-hacc280m lidar500m}; do
  for i in 1 2; do
    for lib in paper_2508_10305_b200/_gpzb.so $cand; do
      echo "== $wl $i $lib" >> gpurun_out/${tag}_ab.txt
      GPZB_LIB=$PWD/$lib timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 \
        | python tools/ab_line.py >> gpurun_out/${tag}_ab.txt
    done
  done
done
cat gpurun_out/${tag}_ab.txt
