#!/bin/bash
# round-2 fourth final pass (separate producer warps, P2M quads): smoke, bench line, launch list,
# ncu of the level-6 M2L, sweep, every GPU test
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f4_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/f4_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/f4_bench.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/f4_bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/f4_bench_ref.log
cat > /tmp/one_eval.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import synthgen, paper_1110_2921_b200 as vf
f = synthgen.make("c4")
ev = vf.Evaluator(p=10, depth=6, image_levels=3, sigma=f.sigma, box_lo=f.box_lo, box_len=f.box_len)
pos = torch.from_numpy(f.pos).cuda(); gam = torch.from_numpy(f.gamma).cuda()
v = torch.empty_like(pos); s = torch.empty_like(pos)
for _ in range(2):
    ev.evaluate_into(pos, gam, v, s)
torch.cuda.synchronize()
PY
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/f4_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-accurate > gpurun_out/f4_ncu_launch.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f4_ncu_dram.csv python /tmp/one_eval.py > gpurun_out/f4_ncu_dram.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:m2l_tc_kernel -s 5 -c 1 -o gpurun_out/m2l_f4 python /tmp/one_eval.py > gpurun_out/f4_ncu_m2l.log 2>&1
timeout 1500 python scripts/bench_sweep.py --configs c1 c2 c3 c5 > gpurun_out/f4_sweep.jsonl 2> gpurun_out/f4_sweep.err
timeout ${TEST_TIMEOUT:-2700} python -m pytest tests -m gpu -q -s -rs > gpurun_out/f4_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f4_pytest_gpu.log
