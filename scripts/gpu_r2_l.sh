#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_P2P_CFG=s4" "VFMM_P2P_CFG=s1" > gpurun_out/lbench.log 2>&1
