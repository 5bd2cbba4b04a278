#!/bin/bash
# round 2, session 2: sanity pass on the restored tree (smoke + bench)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s2a_smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/s2a_bench.log 2>&1; echo "rc=$?" >> gpurun_out/s2a_bench.log
