#!/bin/bash
# full round-2 GPU pass: all GPU tests, the driver-style bench line, the config sweep with
# parity numbers, and the ncu launch list of the bench command
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
{ nproc; lscpu | head -20; nvidia-smi; } > gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 1200 python scripts/bench_sweep.py --configs ${SWEEP:-c1 c2 c3} > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-accurate > gpurun_out/ncu_launch.log 2>&1
timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q -s -rs ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
