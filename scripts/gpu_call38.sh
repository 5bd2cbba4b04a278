#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_A.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_A.log
timeout 600 python -m pytest tests -m gpu -q -x -k "near or fmm_vs_fmm or c4" > gpurun_out/pytest_A.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_A.log
cp var/libvfmm_B.so paper_1110_2921_b200/lib/libvfmm.so
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_B.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_B.log
