#!/bin/bash
# Full GPU tests + hacc and lidar benches + launch lists + one ncu capture.
#   tools/gpu_full.sh <tag> [kernel-regex] [launch-skip] [ncu workload]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1; kre=${2:-^k_encode_dense$}; skip=${3:-0}; nw=${4:-hacc280m}
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
for w in hacc280m lidar500m; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_bench_$w.json 2>> gpurun_out/${tag}_bench.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_$w.csv \
      python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 -o /tmp/${tag}_prof -f \
    python bench.py --workload $nw --steps 1 --warmup 1 --no-e2e --no-cpu --per-call --compress-only > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}_prof.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
ls -la gpurun_out | grep $tag
