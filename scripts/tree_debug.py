"""Debug dump for the treecode: outputs with the P2P / M2P terms dropped (VFMM_TREE_DBG)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthgen
import paper_1110_2921_b200 as vf
f = synthgen.clustered(600)
out = {}
for dbg in ("0", "1", "2"):
    os.environ["VFMM_TREE_DBG"] = dbg
    ev = vf.Evaluator(p=10, depth=4, image_levels=0, sigma=f.sigma, box_lo=f.box_lo, box_len=f.box_len)
    pos = torch.from_numpy(f.pos).cuda(); gam = torch.from_numpy(f.gamma).cuda()
    v, s = ev.evaluate_tree(pos, gam, 0.5, 16)
    torch.cuda.synchronize()
    out["v" + dbg] = v.cpu().numpy(); out["s" + dbg] = s.cpu().numpy()
    ev.close()
np.savez("gpurun_out/tree_debug2.npz", **out)
print("ok")
