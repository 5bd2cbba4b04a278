#!/bin/bash
# tcgen05 M2L after the warp-wide issue: operator stages (AST3 needs XT = 8), XT = 8 alone
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_XT=8" "VFMM_M2L_XT=8 VFMM_M2L_AST3=1" "VFMM_M2L_DBG=2" "VFMM_M2L_DBG=1" "VFMM_M2L_DBG=4" > gpurun_out/ast3_phase.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --p 13 --variants "" "VFMM_M2L_XT=8" >> gpurun_out/ast3_phase.log 2>&1
