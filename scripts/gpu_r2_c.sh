#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_reinit.py tests/test_gpu_parity.py -q -s -k "reinit or engines or tensor_core" > gpurun_out/reinit.log 2>&1; echo "rc=$?" >> gpurun_out/reinit.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
