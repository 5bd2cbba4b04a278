#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "tensor_core_matches or golden" > gpurun_out/g.log 2>&1; echo "rc=$?" >> gpurun_out/g.log
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_DEEP=1" > gpurun_out/deep.log 2>&1
timeout 900 python scripts/bench_sweep.py --configs c5 c2 > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep.err
