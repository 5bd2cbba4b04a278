#!/bin/bash
# tcgen05 M2L with separate operator / window producer warps; P2M strengths loaded once per quad
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_CHAIN=1" > gpurun_out/prod2_phase.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --p 13 --variants "" >> gpurun_out/prod2_phase.log 2>&1
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
PY
VFMM_M2L_DBG=24 timeout 300 python /tmp/tr.py > gpurun_out/prod2_trace.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -s -k "order_split or fmm_vs_fmm or tensor_core or engines or golden or coresident or logical or stage" > gpurun_out/prod2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/prod2_pytest.log
