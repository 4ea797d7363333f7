#!/bin/bash
# Round evidence: tests, smoke, bench, ncu launch list of the bench command,
# one ncu --set full capture of the forward kernel (n=16K), microbenchmarks.
TAG=${1:-round1}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fwd_tc -s 1 -c 1 -o gpurun_out/prof_tc16k_$TAG python tools/prof_tc.py > gpurun_out/ncu_tc_$TAG.log 2>&1
timeout 300 python tools/time_tc.py > gpurun_out/tc_time_$TAG.txt 2>&1
D=128 timeout 300 python tools/time_tc.py > gpurun_out/tc_time_d128_$TAG.txt 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fwd_f32 -s 2 -c 1 -o gpurun_out/prof_fwd16k_$TAG python tools/prof_fwd.py --n 16384 --reps 3 > gpurun_out/ncu_full_$TAG.log 2>&1
./tools/microbench/ffma_variants > gpurun_out/ffma_variants_$TAG.log 2>&1

timeout 300 python tools/time_wide.py 16384 5 > gpurun_out/time_wide_$TAG.txt 2>&1
timeout 300 python bench.py --dist-path --steps 5 --no-sweep --no-cpu-baseline > gpurun_out/bench_distpath_$TAG.log 2>&1
echo done
