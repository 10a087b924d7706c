#!/bin/bash
# B11 fused into the band launch: loopback / peer / slab tests, checked build, halo bench, kbench, bench.
tag=${1:-r2s3h}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_invariants_gpu.py tests/test_parity_full_gpu.py -k "loopback or peer or slab" -x -q > gpurun_out/pytest_fused_$tag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fused_$tag.log
timeout 300 python -m pytest tests/test_checked_build_gpu.py tests/test_trajectory_gpu.py tests/test_nccl_gpu.py -x -q >> gpurun_out/pytest_fused_$tag.log 2>&1; echo "pytest2 exit $?" >> gpurun_out/pytest_fused_$tag.log
timeout 600 python tools/halo_bench.py > gpurun_out/halo_bench_$tag.jsonl 2> gpurun_out/halo_bench_$tag.err
for c in 3 4 5; do timeout 300 python tools/kbench.py --config $c >> gpurun_out/kbench_$tag.log 2>&1; done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo done
