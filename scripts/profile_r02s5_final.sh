#!/bin/bash
# Round-2 session-5 profiling bundle (run under gpurun). Outputs into gpurun_out/r02p_*.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
O=gpurun_out/r02s5fin
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > ${O}_gpu.txt 2>&1
# 1. driver-like bench lines (both arms) + c3 workload
timeout 1200 python bench.py --steps 20 --warmup 5 > ${O}_bench_c2.log 2>&1; echo "bench c2 rc=$?"
timeout 1200 python bench.py --workload c3 --steps 2 --warmup 3 --no-cpu-baseline > ${O}_bench_c3.log 2>&1; echo "bench c3 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > ${O}_bench_ref.log 2>&1; echo "bench ref rc=$?"
# 2. ncu launch list of ONE timed bench step (LPS launches per step, 3 warm-up steps first)
LPS=$(python -c "import json;d=json.loads([x for x in open('${O}_bench_c2.log') if x.startswith('{')][-1]);print(int(d['gpu_launches']/d['steps']))")
echo "LPS=$LPS"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * LPS)) -c $LPS --csv --log-file ${O}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > ${O}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python scripts/launch_summary.py ${O}_launches.csv 25 > ${O}_launches_summary.txt 2>&1
# 3. ncu --set full captures: tridiagonalisation (both C2 sizes), IPT colour, K9 fused epilogue
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sytrd_smem -s 2 -c 2 -o ${O}_sytrd_full python scripts/bench_eig.py 1 1080x270 1920x480 > ${O}_ncu_sytrd.log 2>&1; echo "ncu sytrd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_color_u8 -c 2 -o ${O}_color_full python scripts/bench_elementwise.py 1 c2 > ${O}_ncu_color.log 2>&1; echo "ncu color rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_small_ttm2_resid -c 1 -o ${O}_k9_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > ${O}_ncu_k9.log 2>&1; echo "ncu k9 rc=$?"
for r in sytrd_full color_full k9_full; do
  ncu -i ${O}_${r}.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum > ${O}_${r}_raw.csv 2>&1
done
# 4. every BASELINE config end to end on one GPU + kernel families for C4/C5
timeout 1500 python scripts/run_configs.py c1 c3 c4_8 c4_4 c4_2 c5 > ${O}_configs.txt 2>&1; echo "configs rc=$?"
timeout 900 python scripts/config_families.py c5 c4_2 > ${O}_families.txt 2>&1; echo "families rc=$?"
# 5. row-sharded C5 (2 thread-ranks on one GPU), 2 sweeps
timeout 900 python scripts/run_sharded_emulated.py c5 2 2 > ${O}_sharded_c5.txt 2>&1; echo "sharded rc=$?"
tail -2 ${O}_bench_c2.log | cut -c1-400
