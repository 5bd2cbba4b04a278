#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for v in base V1 V2 V3; do
cp var/libvfmm_$v.so paper_1110_2921_b200/lib/libvfmm.so
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v.log 2>&1
echo "$v $(grep -o '"p2p": [0-9.]*' gpurun_out/bench_$v.log)" >> gpurun_out/variants.log
done
