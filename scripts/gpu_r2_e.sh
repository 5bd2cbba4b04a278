#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -s -x -k "north_star or engines or fmm_vs_fmm or tensor_core" > gpurun_out/p13.log 2>&1; echo "rc=$?" >> gpurun_out/p13.log
timeout 900 python scripts/phase_bench.py --config c4 --p 13 --variants "" "VFMM_M2L=simt" > gpurun_out/p13bench.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --p 12 --variants "" > gpurun_out/p12bench.log 2>&1
