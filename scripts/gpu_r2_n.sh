#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "near_only or dense or clustered or golden or coresident" > gpurun_out/n.log 2>&1; echo "rc=$?" >> gpurun_out/n.log
timeout 900 python scripts/phase_bench.py --config c4 --variants "" > gpurun_out/nbench.log 2>&1
