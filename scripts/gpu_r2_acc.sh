cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for a in "--n 16 --depth 2 --p 10 --lam 1" "--n 32 --depth 3 --p 10 --lam 1" "--n 32 --depth 3 --p 6 --lam 3" "--n 64 --depth 4 --p 8 --lam 1"; do
  echo "== $a" >> gpurun_out/acc.log
  timeout 900 python scripts/m2l_tc_accuracy.py $a >> gpurun_out/acc.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -k "tensor_core or dense" > gpurun_out/tc.log 2>&1
