#!/bin/bash
# order-split M2L (VFMM_M2L_SPLIT) accuracy + timing; L2P two-particle kernel A/B; parity subset
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 200 python scripts/m2l_tc_accuracy.py --n 32 --depth 3 --p 10 > gpurun_out/split_tcacc.log 2>&1
VFMM_M2L_SPLIT=full timeout 200 python scripts/m2l_tc_accuracy.py --n 32 --depth 3 --p 10 >> gpurun_out/split_tcacc.log 2>&1
timeout 200 python scripts/m2l_tc_accuracy.py --n 32 --depth 3 --p 13 >> gpurun_out/split_tcacc.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_SPLIT=full" "VFMM_M2L_SPLIT=5" "VFMM_M2L_SPLIT=7" "VFMM_L2P=single" > gpurun_out/split_phase.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --p 13 --variants "" "VFMM_M2L_SPLIT=full" "VFMM_M2L_SPLIT=5" >> gpurun_out/split_phase.log 2>&1
timeout 1200 python scripts/m2l_split_accuracy.py > gpurun_out/split_acc.jsonl 2> gpurun_out/split_acc.err
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "tensor_core or golden or p_sweep or fmm_vs_fmm or clustered or north_star" > gpurun_out/split_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/split_pytest.log
