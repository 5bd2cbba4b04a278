#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_reinit.py -q -s > gpurun_out/reinit.log 2>&1; echo "rc=$?" >> gpurun_out/reinit.log
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_P2P_CFG=b3u1" "VFMM_P2P_CFG=b3u2" "VFMM_P2P_CFG=b2u1" "VFMM_P2P=sj" > gpurun_out/p2pvar.log 2>&1
