#!/bin/bash
# round 2: tables built from kernel-parameter bases + entry prefetch (scan launch
# cost), restore/checkpoint fenced after caller work; all GPU tests, racecheck
# re-run, K8 stamps, bench (compress on = default, and off)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2f_smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2f_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2f_gputests.log
GCR_SCAN_TIMES=1 timeout 300 python tools/scan_times.py 128 1024 4096 > gpurun_out/r2f_scan_times.log 2>&1
timeout 600 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
timeout 600 python bench.py --compress 0 --no-cpu-baseline > gpurun_out/r2f_bench_plain.json 2> gpurun_out/r2f_bench_plain.err
SEL="tests/test_gpu_parity.py::test_c1_full_parity_and_round_trip tests/test_gpu_parity.py::test_page_sizes_tails_and_zero_pages[4096-0] tests/test_gpu_parity.py::test_page_sizes_tails_and_zero_pages[65536-18446744073709551615] tests/test_gpu_parity.py::test_page_sizes_tails_and_zero_pages[2097152-1048576] tests/test_gpu_parity.py::test_chunking_and_copy_streams[1048576-2-262144] tests/test_gpu_parity.py::test_incremental_chain_parity[4096-0] tests/test_gpu_verify.py::test_verify_counts_and_first_bad_match_oracle[0-2097152-4194304] tests/test_gpu_codec.py::test_compressed_stream_equals_oracle_and_restores[65536-1048576] tests/test_gpu_codec.py::test_compressed_incremental_chain[4096]"
for tool in racecheck memcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python -m pytest -q -m gpu -p no:cacheprovider $SEL > gpurun_out/r2f_sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2f_sanitizer_$tool.log
done
