#!/bin/bash
# round-2 first GPU check: bench arms (c2, c3, reference), GPU tests
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nproc > gpurun_out/r02_nproc.txt; lscpu | head -20 >> gpurun_out/r02_nproc.txt
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_c2.log 2>&1; echo "c2 rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r02_bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --workload c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c3.log 2>&1; echo "c3 rc=$?"
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_pytest_gpu.log
