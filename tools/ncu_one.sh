#!/bin/bash
# ncu --set full of one kernel launch of the bench (per-call mode):
#   tools/ncu_one.sh <tag> <kernel-regex> <launch-skip> [extra bench args]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; kre=$2; skip=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c ${NCU_COUNT:-1} -o /tmp/${tag}_prof -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --per-call "$@" > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}_prof.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
ls -la gpurun_out | grep $tag
