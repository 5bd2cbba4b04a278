#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "fmm_vs_fmm or deterministic or 27cubed_images or (engines and not 64-5)" > gpurun_out/h.log 2>&1; echo "rc=$?" >> gpurun_out/h.log
timeout 900 python scripts/phase_bench.py --config c4 --variants "" > gpurun_out/hbench.log 2>&1
