#!/bin/bash
# TMA bulk-copy vs vector-copy microbenchmark (64 KiB pieces, permuted);
# restore timeline A/B (region ring vs slot-per-stream) on one box
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2v_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_copy/tma_copy tools/tma_copy/tma_copy.cu
timeout 300 tools/tma_copy/tma_copy 1024 > gpurun_out/r2v_tma_copy_1g.jsonl 2>&1
timeout 300 tools/tma_copy/tma_copy 4096 > gpurun_out/r2v_tma_copy_4g.jsonl 2>&1
for k in 1 2; do for R in 1 0; do
GCR_RESTORE_RING=$R GCR_TRACE=1 timeout 300 python tools/restore_timing.py 65536 > gpurun_out/r2v_rt_ring${R}_$k.log 2> gpurun_out/r2v_rt_ring${R}_$k.err
done; done
timeout 900 python -m pytest tests/test_gpu_codec.py -m gpu -q -k ring > gpurun_out/r2v_tests.log 2>&1; echo rc=$? >> gpurun_out/r2v_tests.log
