#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for v in cur H1 H2; do
for m in cross sj; do
cp var/libvfmm_$v.so paper_1110_2921_b200/lib/libvfmm.so
VFMM_P2P=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$v$m.log 2>&1
echo "$v $m $(grep -o '"p2p": [0-9.]*' gpurun_out/bench_$v$m.log)" >> gpurun_out/variants.log
done
done
cp var/libvfmm_H1.so paper_1110_2921_b200/lib/libvfmm.so
timeout 600 python -m pytest tests -m gpu -q -x -k "near or fmm_vs_fmm or c4" > gpurun_out/pytest_H1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_H1.log
