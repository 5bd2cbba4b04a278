#!/bin/bash
# ncu captures for round 2: (1) per-kernel duration + DRAM bytes of one c4 evaluation
# (the HBM roofline table), (2) full set with source of the P2P kernel, (3) full set of the
# level-6 tcgen05 M2L launch
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
cat > /tmp/one_eval.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import synthgen, paper_1110_2921_b200 as vf
f = synthgen.make("c4")
ev = vf.Evaluator(p=10, depth=6, image_levels=3, sigma=f.sigma, box_lo=f.box_lo, box_len=f.box_len)
pos = torch.from_numpy(f.pos).cuda(); gam = torch.from_numpy(f.gamma).cuda()
v = torch.empty_like(pos); s = torch.empty_like(pos)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    ev.evaluate_into(pos, gam, v, s)
torch.cuda.synchronize()
PY
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_dram.csv python /tmp/one_eval.py 2 > gpurun_out/ncu_dram.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:p2p_kernel -s 1 -c 1 -o gpurun_out/p2p_full python /tmp/one_eval.py 2 > gpurun_out/ncu_p2p.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:m2l_tc_kernel -s 5 -c 1 -o gpurun_out/m2l_full python /tmp/one_eval.py 2 > gpurun_out/ncu_m2l.log 2>&1
ls -la gpurun_out
