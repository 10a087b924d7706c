#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, launch list and one ncu --set full capture of the
# stage kernel (summarised on the box; the .ncu-rep stays in /tmp there).
# Usage (from the repo root, on the GPU box): bash tools/gpu_check.sh [tag]
tag=${1:-r1}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
for c in 3 4 5 2 1; do timeout 300 python tools/kbench.py --config $c >> gpurun_out/kbench_$tag.log 2>&1; done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain_$tag.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 4 -c 2 -o /tmp/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1
if [ -f /tmp/prof_$tag.ncu-rep ]; then
  python tools/ncu_summary.py /tmp/prof_$tag.ncu-rep > gpurun_out/ncu_summary_$tag.txt 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$tag.csv 2>/dev/null
  ncu -i /tmp/prof_$tag.ncu-rep --page details > gpurun_out/ncu_details_$tag.txt 2>/dev/null
  ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_$tag.csv 2>/dev/null
fi
echo done
