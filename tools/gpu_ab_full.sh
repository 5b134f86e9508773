#!/bin/bash
# Full GPU tests + smoke with the in-tree library, then the in-tree library
# against every build/*.so (tools/gpu_ab_multi.sh).   tools/gpu_ab_full.sh <tag>
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
tag=$1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.txt
tail -n 2 gpurun_out/${tag}_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.txt
WLS="${WLS:-hacc280m decomp1b}" R=${R:-2} bash tools/gpu_ab_multi.sh $tag
