#!/bin/bash
# tcgen05 M2L: offsets per full-split TMEM chain (VFMM_M2L_CHAIN = 1, 2, 3): time and accuracy
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_CHAIN=2" "VFMM_M2L_CHAIN=3" > gpurun_out/chain_phase.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --p 13 --variants "" "VFMM_M2L_CHAIN=2" "VFMM_M2L_CHAIN=3" >> gpurun_out/chain_phase.log 2>&1
for c in 2 3; do
VFMM_M2L_CHAIN=$c timeout 1500 python -m pytest tests/test_gpu_parity.py -q -s -k "tensor_core or engines or order_split or golden" > gpurun_out/chain${c}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/chain${c}_pytest.log
done
