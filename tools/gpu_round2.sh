#!/bin/bash
# Round-2 evidence run: GPU tests, smoke, the bench line (+ reference arm and
# the other workloads), the ncu launch list, per-call traffic and --set full
# captures of the top kernels (raw + source pages as CSV).
#   tools/gpu_round2.sh <tag>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/${tag}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/${tag}_bench_n1.json 2> gpurun_out/${tag}_bench_n1.err
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
for w in lidar500m decomp1b snapshot2b; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu > gpurun_out/${tag}_bench_$w.json 2> gpurun_out/${tag}_bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
for w in hacc280m lidar500m; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${tag}_traffic_$w.csv python bench.py --workload $w --per-call --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
cap() {  # name regex skip [extra bench args]
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 1 -o /tmp/${tag}_$1 -f \
      python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --per-call $4 > gpurun_out/${tag}_$1_ncu.log 2>&1
  ncu -i /tmp/${tag}_$1.ncu-rep --page raw --csv > gpurun_out/${tag}_$1_raw.csv 2>/dev/null
  ncu -i /tmp/${tag}_$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_$1_src.csv 2>/dev/null
}
cap k2s_vel "^k_encode_small" 2 --compress-only
cap k2p_pos "^k_encode_warp" 1 --compress-only  # launch 0 is the list variant of the position call, which exits
cap k4w_vel "^k_decode_warp" 1
cap k1_range "^k_range_w" 0 --compress-only
cap k3b_vel "^k_copy_payloads" 1 --compress-only
ls -la gpurun_out | grep $tag
