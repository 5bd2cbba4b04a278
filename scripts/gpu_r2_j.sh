#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sigma.py tests/test_gpu_dist.py -q -s -x -k "near_only or dense or clustered or fmm_vs_fmm or golden or direct_mode or deterministic or sigma or logical or coresident" > gpurun_out/j.log 2>&1; echo "rc=$?" >> gpurun_out/j.log
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_P2P=cross" > gpurun_out/jbench.log 2>&1
