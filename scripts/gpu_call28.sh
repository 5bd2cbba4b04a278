#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p_kernel -c 1 -o gpurun_out/p2p_sj python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_p2p.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_p2p.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_tc_kernel -c 1 -o gpurun_out/m2ltc2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_m2l.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_m2l.log
