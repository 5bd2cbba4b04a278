#!/bin/bash
# tcgen05 M2L timeline (chains across groups, split producers) with loads / drain removed
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
cat > /tmp/tr.py <<'PY'
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
print("m2l", ev.stats()["ms_m2l"])
PY
for d in 24 26 30 31; do VFMM_M2L_DBG=$d timeout 300 python /tmp/tr.py > gpurun_out/tr4_$d.log 2>&1; done
