#!/bin/bash
# round-2 eighth final pass (HEAD): every GPU test
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/f8_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f8_pytest_gpu.log
