#!/bin/bash
# round-2 seventh final pass (HEAD): smoke, bench line, parity at the bench configuration, treecode tests
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f7_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f7_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f7_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/f7_bench.log
timeout 1200 python -m pytest tests/test_gpu_tree.py tests/test_gpu_parity.py -q -s -k "tree or hybrid or golden or c1_fmm or near_only" > gpurun_out/f7_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f7_pytest.log
