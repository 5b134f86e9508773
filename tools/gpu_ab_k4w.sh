#!/bin/bash
# K4w A/B: decode parity tests with build/<cand>.so, then every build/*.so
# against the in-tree library (tools/gpu_ab_multi.sh).
#   tools/gpu_ab_k4w.sh <tag> <cand>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; cand=build/$2.so
GPZB_LIB=$PWD/$cand timeout 900 python -m pytest tests -x -q -m gpu -k "decode or decompress or golden or bitflip or streamed or iter or warp or stress or bench_workload or configs" > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
tail -n 2 gpurun_out/${tag}_pytest.txt
WLS="${WLS:-hacc280m decomp1b}" R=${R:-2} bash tools/gpu_ab_multi.sh $tag
