#!/bin/bash
# round 2: codec page slicing (large pages get several warps) + K6 back to the
# vector copy: codec/parity tests, restore host-cost timing, C2 2 MiB / 4 KiB /
# 64 KiB compressed and staged benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2o_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_codec.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2o_tests.log 2>&1; echo rc=$? >> gpurun_out/r2o_tests.log
timeout 300 python tools/restore_timing.py 4096 > gpurun_out/r2o_restore_timing_4k.log 2>&1
timeout 300 python tools/restore_timing.py 2097152 > gpurun_out/r2o_restore_timing_2m.log 2>&1
for P in 2097152 4096 65536; do
  timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --page-size $P --steps 5 > gpurun_out/r2o_bench_$P.json 2> gpurun_out/r2o_bench_$P.err
done
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --direct-min-mb -1 --steps 5 > gpurun_out/r2o_bench_staged.json 2> gpurun_out/r2o_bench_staged.err
