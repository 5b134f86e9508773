"""Print the A/B bench lines of tools/gpu_ab_lib.sh: python tools/ab_show.py <tag>"""
import glob
import json
import sys

tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{tag}_*[0-9].json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f"{f:40s} compress {d['ms_per_step']:.3f} ms ({d['value']:.0f} GB/s)  "
              f"decompress {d['decompress']['ms_per_step']:.3f} ms ({d['decompress']['value']:.0f} GB/s)")
    except Exception as e:  # noqa: BLE001
        print(f, "?", e)
