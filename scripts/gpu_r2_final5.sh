#!/bin/bash
# round-2 fifth final pass (treecode + hybrid): smoke, tree tests and timings, an ncu capture of
# the treecode kernel, bench line + reference arm, launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f5_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f5_smoke.log
timeout 900 python -m pytest tests/test_gpu_tree.py -q -s > gpurun_out/f5_tree.log 2>&1; echo "rc=$?" >> gpurun_out/f5_tree.log
for a in "--config c2" "--config c3" "--clustered 1000000 --lam 1" "--clustered 1000000 --lam 1 --theta 0.7"; do
  timeout 300 python scripts/tree_bench.py $a --p 10 >> gpurun_out/f5_tree_vs_fmm.jsonl 2>> gpurun_out/f5_tree_vs_fmm.err
done
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f5_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/f5_bench.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/f5_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/f5_bench_ref.log
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/f5_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-accurate > gpurun_out/f5_ncu_launch.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:tree_kernel -c 1 -o gpurun_out/tree_f5 python scripts/tree_bench.py --config c2 --p 10 --reps 1 > gpurun_out/f5_ncu_tree.log 2>&1
