#!/bin/bash
# round 2: f4 codec GPU tests (parity with the oracle, full-size C2/C3), the
# racecheck diagnostic, and bench A/B of compress 0/1 on C2 and C3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2d_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_codec.py -q -m gpu -x > gpurun_out/r2d_codec_tests.log 2>&1; echo rc=$? >> gpurun_out/r2d_codec_tests.log
for P in 65536 2097152; do
  timeout 300 compute-sanitizer --tool racecheck python tools/racecheck_diag.py $P > gpurun_out/r2d_racecheck_diag_$P.log 2>&1
  timeout 300 python tools/racecheck_diag.py $P > gpurun_out/r2d_plain_diag_$P.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --compress 1 > gpurun_out/r2d_bench_c2_compress.json 2> gpurun_out/r2d_bench_c2_compress.err
timeout 600 python bench.py --no-cpu-baseline --compress 0 > gpurun_out/r2d_bench_c2_plain.json 2> gpurun_out/r2d_bench_c2_plain.err
timeout 900 python bench.py --no-cpu-baseline --config C3 --steps 3 --compress 1 > gpurun_out/r2d_bench_c3_compress.json 2> gpurun_out/r2d_bench_c3_compress.err
