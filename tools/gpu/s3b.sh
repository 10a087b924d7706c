#!/bin/bash
# B11 peer-store halo transport: loopback tests, the NCCL test (self-skips on 1 GPU), halo bench.
tag=${1:-r2s3b}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_invariants_gpu.py -k "peer or loopback" -x -q > gpurun_out/pytest_peer_$tag.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_peer_$tag.log
timeout 300 python -m pytest tests/test_nccl_gpu.py tests/test_checked_build_gpu.py -q >> gpurun_out/pytest_peer_$tag.log 2>&1; echo "pytest2 exit $?" >> gpurun_out/pytest_peer_$tag.log
timeout 600 python tools/halo_bench.py > gpurun_out/halo_bench_$tag.jsonl 2> gpurun_out/halo_bench_$tag.err
timeout 300 python tools/halo_bench.py --config 5 --steps 50 > gpurun_out/halo_bench_cfg5_$tag.jsonl 2>> gpurun_out/halo_bench_$tag.err
echo done
