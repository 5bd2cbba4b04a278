#!/bin/bash
# M2L bottleneck probes (VFMM_M2L_DBG: wrong results, timing only) + order-split tests
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_SPLIT=full" "VFMM_M2L_SPLIT=1" "VFMM_M2L_DBG=1" "VFMM_M2L_DBG=2" "VFMM_M2L_DBG=4" "VFMM_M2L_DBG=6" "VFMM_M2L_DBG=7" "VFMM_M2L_SPLIT=1 VFMM_M2L_DBG=1" "VFMM_M2L_SPLIT=full VFMM_M2L_DBG=1" "VFMM_M2L_SPLIT=full VFMM_M2L_DBG=6" > gpurun_out/probe_phase.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -s -k "order_split or fmm_vs_fmm or tensor_core or engines or golden or north_star" > gpurun_out/split2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/split2_pytest.log
