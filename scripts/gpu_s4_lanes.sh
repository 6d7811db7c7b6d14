#!/bin/bash
# C3 lanes A/B: parity test for lanes, then the C3 bench with 1, 2 and 3 lanes.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "encode_stacks" > gpurun_out/s4_lanes_test.log 2>&1; echo "test rc $?" >> gpurun_out/s4_lanes_test.log
for nl in 1 2 3; do
  timeout 900 python bench.py --workload c3 --steps 1 --warmup 3 --lanes $nl --no-cpu-baseline > gpurun_out/s4_c3_l$nl.json 2> gpurun_out/s4_c3_l$nl.err
done
