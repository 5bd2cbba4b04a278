#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
./examples/vfmm_c_example 16 > gpurun_out/c_example.txt 2>&1; echo "rc=$?" >> gpurun_out/c_example.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c_example" > gpurun_out/pytest_tc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc.log
