#!/bin/bash
# round 2: bench line (N=1), 2 ranks on the 1-GPU box (launch plumbing), the
# reference arm (whole C2), C4 1% incremental, and compute-sanitizer
# memcheck / racecheck / synccheck over small parity cases (K1, K1g, multi-chunk,
# staged and direct drains, restore scatter + zero fill + verify)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2c_build.log 2>&1
timeout 600 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 600 python bench.py --gpus 2 --steps 5 --no-cpu-baseline > gpurun_out/r2c_bench_2ranks.json 2> gpurun_out/r2c_bench_2ranks.err
timeout 600 python bench.py --impl reference > gpurun_out/r2c_bench_ref.json 2> gpurun_out/r2c_bench_ref.err
timeout 600 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --no-cpu-baseline > gpurun_out/r2c_c4_inc1.json 2> gpurun_out/r2c_c4_inc1.err
SEL="tests/test_gpu_parity.py::test_c1_full_parity_and_round_trip tests/test_gpu_parity.py::test_page_sizes_tails_and_zero_pages[4096-0] tests/test_gpu_parity.py::test_page_sizes_tails_and_zero_pages[65536-18446744073709551615] tests/test_gpu_parity.py::test_page_sizes_tails_and_zero_pages[2097152-1048576] tests/test_gpu_parity.py::test_chunking_and_copy_streams[1048576-2-262144] tests/test_gpu_parity.py::test_incremental_chain_parity[4096-0] tests/test_gpu_verify.py::test_verify_counts_and_first_bad_match_oracle[0-2097152-4194304]"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 python -m pytest -q -m gpu -p no:cacheprovider $SEL > gpurun_out/r2c_sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r2c_sanitizer_$tool.log
done
