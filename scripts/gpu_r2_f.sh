#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "tensor_core_matches or coresident or north_star" > gpurun_out/fix.log 2>&1; echo "rc=$?" >> gpurun_out/fix.log
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_CORES=1" > gpurun_out/cores.log 2>&1
timeout 900 python scripts/phase_bench.py --config c4 --p 13 --variants "" "VFMM_CORES=1" >> gpurun_out/cores.log 2>&1
timeout 1200 python scripts/bench_sweep.py --configs c3 > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep.err
