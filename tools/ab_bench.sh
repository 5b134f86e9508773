#!/bin/bash
# A/B: bench the default build and every build/*.so variant (compress/decompress GB/s only)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for lib in paper_2508_10305_b200/_gpzb.so $(ls build/*.so 2>/dev/null); do
  echo "== $lib" >> gpurun_out/ab.txt
  GPZB_LIB=$PWD/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu $AB_ARGS 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    pd=d['kernels']['per_dataset_ms']; f=lambda v: '/'.join('%.3f' % x if x else '-' for x in v)
    print('comp %.1f decomp %.1f k_encode %s k_decode %s k_range %.3f cr %.3f clk %s' % (d['value'], d['decompress']['value'], f(pd['k_encode']), f(pd['k_decode']), d['kernels']['k_range_ms'], d['compression_ratio'], d['clocks']['sm_mhz'] if d['clocks'] else None))
" >> gpurun_out/ab.txt
done
cat gpurun_out/ab.txt
