"""Per-phase timing probe: run c4 a few times, print library phase events (and a variant
with a host sync between phases, VFMM_DEBUG_SYNC)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthgen
import paper_1110_2921_b200 as vf
f = synthgen.make("c4")
ev = vf.Evaluator(p=10, depth=6, image_levels=3, sigma=f.sigma, box_lo=f.box_lo, box_len=f.box_len)
pos = torch.from_numpy(f.pos).cuda(); gam = torch.from_numpy(f.gamma).cuda()
for i in range(4):
    ev.evaluate(pos, gam)
    torch.cuda.synchronize()
    s = ev.stats()
    print({k: round(v, 3) for k, v in s.items() if k.startswith("ms_")}, flush=True)
