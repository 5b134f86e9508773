"""Build the library with extra nvcc -D flags into build/<name>.so (A/B candidates):
python tools/build_variant.py <name> [-DFOO=1 ...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as g  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
out = os.path.join(ROOT, "build", name + ".so")
subprocess.run([g._nvcc(), *g.NVCC_FLAGS, *defs, "-o", out, os.path.join(g.CSRC, "gpzb_capi.cu")], check=True)
usage = subprocess.run(["cuobjdump", "--dump-resource-usage", out], capture_output=True, text=True).stdout
lines = usage.splitlines()
for i, l in enumerate(lines):
    if "Function" in l and any(k in l for k in sys.argv[2:3] and [] or ["decode_warp", "encode_small", "encode_warp"]):
        print(l.strip()[:90], "|", lines[i + 1].strip()[:120])
