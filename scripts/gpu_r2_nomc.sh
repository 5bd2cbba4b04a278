#!/bin/bash
# tcgen05 M2L: operator multicast vs each CTA loading its own operators (VFMM_M2L_NOMC=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_NOMC=1" "VFMM_M2L_NOMC=1 VFMM_M2L_XT=8 VFMM_M2L_AST3=1" > gpurun_out/nomc_phase.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --p 13 --variants "" "VFMM_M2L_NOMC=1" >> gpurun_out/nomc_phase.log 2>&1
VFMM_M2L_NOMC=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -s -k "tensor_core or order_split or golden" > gpurun_out/nomc_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/nomc_pytest.log
