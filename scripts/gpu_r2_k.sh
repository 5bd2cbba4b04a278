#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
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
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:p2p_kernel -s 1 -c 1 -o gpurun_out/p2p_box_full python /tmp/one_eval.py > gpurun_out/ncu_p2p.log 2>&1
