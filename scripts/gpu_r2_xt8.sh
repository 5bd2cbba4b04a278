#!/bin/bash
# tcgen05 M2L: XT = 8 / T = 8 slab layout (240-row windows) and a third operator stage
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_XT=8" "VFMM_M2L_XT=8 VFMM_M2L_AST3=1" > gpurun_out/xt8_phase.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --p 13 --variants "" >> gpurun_out/xt8_phase.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -s -k "order_split or fmm_vs_fmm or tensor_core or engines or golden or coresident or logical" > gpurun_out/xt8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/xt8_pytest.log
VFMM_M2L_XT=8 VFMM_M2L_AST3=1 timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -s -k "order_split or tensor_core or golden" > gpurun_out/xt8_pytest2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/xt8_pytest2.log
