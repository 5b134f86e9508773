#!/bin/bash
# Round-2 state check: GPU tests, smoke, bench of every workload, launch list,
# traffic per kernel, one ncu --set full capture of the velocity encoder.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-r02s}; kre=${2:-^k_encode_small}; skip=${3:-0}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_gpu.txt
timeout 1500 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --per-call --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/${tag}_bench_pc.json 2>> gpurun_out/${tag}_bench.err
for w in lidar500m decomp1b snapshot2b; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_traffic_hacc.csv python bench.py --per-call --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 -o /tmp/${tag}_prof -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --per-call --compress-only > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}_prof.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_src.csv 2>/dev/null
ls -la gpurun_out | grep $tag
