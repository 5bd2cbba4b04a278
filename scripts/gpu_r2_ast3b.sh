#!/bin/bash
# tcgen05 M2L after the producer split: a third operator stage (XT = 8 layout)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_XT=8" "VFMM_M2L_XT=8 VFMM_M2L_AST3=1" "VFMM_M2L_XT=8 VFMM_M2L_AST3=1 VFMM_M2L_CHAIN=1" > gpurun_out/ast3b_phase.log 2>&1
