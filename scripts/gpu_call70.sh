#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for cfg in "--config c2" "--config c3" "--config c5" "--depth 5" "--depth 7"; do
timeout 900 python bench.py $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b.log 2>&1
echo "$cfg rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b.log) $(grep -o '"phase_ms": {[^}]*}' gpurun_out/b.log)" >> gpurun_out/configs.log
done
