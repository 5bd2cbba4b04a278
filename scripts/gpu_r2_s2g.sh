#!/bin/bash
# round 2, session 2: hybrid mode choosing n_crit too: the treecode tests
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tree.py -q -s > gpurun_out/s2g_tree.log 2>&1; echo "rc=$?" >> gpurun_out/s2g_tree.log
