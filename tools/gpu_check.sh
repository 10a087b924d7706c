#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, launch list and one ncu --set full capture.
# Usage (from the repo root, on the GPU box): bash tools/gpu_check.sh [tag]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 300 python tools/kbench.py --config 3 > gpurun_out/kbench_$tag.log 2>&1
timeout 300 python tools/kbench.py --config 4 >> gpurun_out/kbench_$tag.log 2>&1
timeout 300 python tools/kbench.py --config 5 >> gpurun_out/kbench_$tag.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_$tag.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 4 -c 2 -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1
echo done
