#!/bin/bash
# compute-sanitizer (racecheck, memcheck, synccheck) over the round-2 paths:
# the TMA scatter ring (default), the TMA pack (GCR_TMA_COPY=2), the restore
# region ring with the speculative prefix (f4), codec; D2H under SM load
# (globaltimer-bounded load kernel, no host polling)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2za_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/d2h_interference/d2h tools/d2h_interference/d2h_interference.cu
timeout 300 tools/d2h_interference/d2h > gpurun_out/r2za_d2h_interference.jsonl 2>&1
SEL="tests/test_gpu_parity.py::test_copy_kernel_variants tests/test_gpu_codec.py::test_restore_region_ring_reuse tests/test_gpu_parity.py::test_c1_full_parity_and_round_trip tests/test_gpu_parity.py::test_page_sizes_tails_and_zero_pages[65536-18446744073709551615] tests/test_gpu_codec.py::test_compressed_stream_equals_oracle_and_restores[65536-1048576] tests/test_gpu_codec.py::test_compressed_incremental_chain[4096]"
for tool in racecheck memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python -m pytest -q -m gpu -p no:cacheprovider $SEL > gpurun_out/r2za_sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2za_sanitizer_$tool.log
done
