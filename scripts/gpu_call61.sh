#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2m_kernel -c 1 -o gpurun_out/p2m_f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_p2m.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:translate_kernel -c 1 -o gpurun_out/m2m_f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_m2m.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:l2p_combine -c 1 -o gpurun_out/l2p_f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_l2p.log 2>&1
