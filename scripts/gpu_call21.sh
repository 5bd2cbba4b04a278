#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
./scripts/micro/fma_pipes > gpurun_out/fma_pipes.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:l2p_combine -c 1 -o gpurun_out/l2p2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l2p.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_l2p.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_tc_kernel -c 1 -o gpurun_out/m2ltc python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_m2l.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_m2l.log
