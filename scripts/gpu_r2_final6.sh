#!/bin/bash
# round-2 sixth final pass (the session's last code: treecode + hybrid): smoke, bench line,
# launch list, every GPU test
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f6_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f6_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/f6_bench.log
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/f6_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-accurate > gpurun_out/f6_ncu_launch.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -s -rs > gpurun_out/f6_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f6_pytest_gpu.log
