#!/bin/bash
# tcgen05 M2L: timeline probe + phase times + parity after the issuer rewrite (merged chains)
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
print("m2l ms", ev.stats()["ms_m2l"])
PY
for v in "VFMM_M2L_DBG=8" "VFMM_M2L_DBG=8 VFMM_M2L_SPLIT=full" "VFMM_M2L_DBG=9"; do
  echo "=== $v" >> gpurun_out/trace2.log
  env $v timeout 300 python /tmp/tr.py 2>&1 | grep -A7 "cta 0" | tail -8 >> gpurun_out/trace2.log
done
timeout 600 python scripts/phase_bench.py --config c4 --variants "" "VFMM_M2L_SPLIT=full" > gpurun_out/trace2_phase.log 2>&1
timeout 600 python scripts/phase_bench.py --config c4 --p 13 --variants "" "VFMM_M2L_SPLIT=full" >> gpurun_out/trace2_phase.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -s -k "order_split or fmm_vs_fmm or tensor_core or engines or golden or north_star" > gpurun_out/trace2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/trace2_pytest.log
