#!/bin/bash
# One gpurun call: smoke, GPU tests, bench, ncu launch list + full capture.
# usage: bash tools/gpu_round.sh [tag] [skip-list: smoke,tests,bench,launches,full]
TAG=${1:-r}
SKIP=${2:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
[[ $SKIP == *smoke* ]] || { timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log; }
[[ $SKIP == *tests* ]] || { timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log; }
[[ $SKIP == *bench* ]] || { timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log; }
[[ $SKIP == *launches* ]] || timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
[[ $SKIP == *full* ]] || timeout 400 ncu --set full --clock-control none --import-source on -k regex:fwd_f32 -s 2 -c 1 -o gpurun_out/prof_fwd16k_$TAG python tools/prof_fwd.py --n 16384 --reps 3 > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
