#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_targets.py -q -s > gpurun_out/step.log 2>&1; echo "rc=$?" >> gpurun_out/step.log
timeout 1200 python scripts/m2l_tc_accuracy.py --n 64 --depth 5 --p 10 --lam 3 > gpurun_out/acc5.log 2>&1
