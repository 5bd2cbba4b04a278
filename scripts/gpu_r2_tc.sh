#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "tensor_core or engines or fmm_vs_fmm or deterministic or 27cubed" > gpurun_out/tc.log 2>&1; echo "rc=$?" >> gpurun_out/tc.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -q -s > gpurun_out/dist.log 2>&1; echo "rc=$?" >> gpurun_out/dist.log
