#!/bin/bash
# one gpurun call: host info, smoke, GPU tests, bench (each under its own timeout)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
{ nproc; lscpu | head -20; nvidia-smi; } > gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
