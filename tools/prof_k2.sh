cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_encode$" -s 3 -c 1 -o /tmp/prof_k2p -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --per-call --compress-only > gpurun_out/ncu_k2.log 2>&1
ncu -i /tmp/prof_k2p.ncu-rep --page source --csv --print-source cuda,sass --launch-skip 0 --launch-count 1 > /tmp/k2p_src.csv 2>/dev/null
python tools/ncu_phase.py /tmp/k2p_src.csv gpzb_encode_narrow.cuh > gpurun_out/k2p_phase.txt 2>&1
python tools/ncu_source_top.py /tmp/k2p_src.csv > gpurun_out/k2p_top.txt 2>&1
ncu -i /tmp/prof_k2p.ncu-rep --page details --csv --launch-skip 0 --launch-count 1 > gpurun_out/k2p_details.csv 2>/dev/null
ls -la /tmp/k2p_src.csv
cp /tmp/k2p_src.csv gpurun_out/k2p_src.csv
