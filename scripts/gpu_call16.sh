#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:l2p_combine -c 1 -o gpurun_out/l2p python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l2p.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_l2p.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:translate_kernel --launch-skip 12 -c 1 -o gpurun_out/l2l python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l2l.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_l2l.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p_kernel -c 1 -o gpurun_out/p2p python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_p2p.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_p2p.log
