# ncu source-level capture of one K4w launch (launch index $1 among k_decode_warp launches)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
s=${1:-2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_decode_warp$" -s $s -c 1 -o /tmp/prof_k4 -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --per-call > gpurun_out/ncu_k4.log 2>&1
ncu -i /tmp/prof_k4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/k4_src.csv 2>/dev/null
ncu -i /tmp/prof_k4.ncu-rep --page details --csv > gpurun_out/k4_details.csv 2>/dev/null
