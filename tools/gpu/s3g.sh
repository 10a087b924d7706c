#!/bin/bash
# both boundary bands in one pair launch (Layout gap): loopback tests, halo bench, checked build.
tag=${1:-r2s3g}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_invariants_gpu.py tests/test_parity_full_gpu.py -k "loopback or peer or slab" -x -q > gpurun_out/pytest_fold_$tag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fold_$tag.log
timeout 300 python -m pytest tests/test_checked_build_gpu.py tests/test_trajectory_gpu.py -x -q >> gpurun_out/pytest_fold_$tag.log 2>&1; echo "pytest2 exit $?" >> gpurun_out/pytest_fold_$tag.log
timeout 600 python tools/halo_bench.py > gpurun_out/halo_bench_$tag.jsonl 2> gpurun_out/halo_bench_$tag.err
echo done
