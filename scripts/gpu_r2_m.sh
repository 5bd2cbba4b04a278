#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sigma.py -q -s -x -k "near_only or dense or clustered or fmm_vs_fmm or golden or direct_mode or sigma or p_sweep or c1_fmm" > gpurun_out/m.log 2>&1; echo "rc=$?" >> gpurun_out/m.log
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_P2P_CFG=s2" "VFMM_P2P=cross" > gpurun_out/mbench.log 2>&1
