#!/bin/bash
# round-2 GPU call: build check, host info, GPU tests (verbose prints), short bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nproc; lscpu | head -20; nvidia-smi; } > gpurun_out/host.txt 2>&1
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -s -rs ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -n "$BENCH" ]; then timeout 900 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3 --no-cpu-baseline} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; fi
