#!/bin/bash
# round 2, session 2: treecode + hybrid tests, then the full GPU suite
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tree.py -q -s > gpurun_out/s2c_tree.log 2>&1; echo "rc=$?" >> gpurun_out/s2c_tree.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/s2c_gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/s2c_gpu_all.log
