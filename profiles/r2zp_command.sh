#!/bin/bash
# round over round on ONE box: round 1's final code (4a6aac6, built in
# tools/ab_r1) vs the current code, alternating: C2 default line (r1: plain;
# now: f4 and plain), C3 (r1 plain, now f4 / plain), C5 16 GiB at 4 KiB, C4 1 %
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2zp_build.log 2>&1
(cd tools/ab_r1 && python -c "import __graft_entry__ as g; g.build()") >> gpurun_out/r2zp_build.log 2>&1
for k in 1 2; do
  (cd tools/ab_r1 && timeout 600 python bench.py --no-cpu-baseline --steps 10 > ../../gpurun_out/r2zp_r1_c2_$k.json 2>/dev/null)
  timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --steps 10 > gpurun_out/r2zp_now_c2_$k.json 2>/dev/null
  timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --steps 10 --compress 0 > gpurun_out/r2zp_now_c2plain_$k.json 2>/dev/null
  (cd tools/ab_r1 && timeout 900 python bench.py --no-cpu-baseline --config C3 --steps 3 > ../../gpurun_out/r2zp_r1_c3_$k.json 2>/dev/null)
  timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C3 --steps 3 > gpurun_out/r2zp_now_c3_$k.json 2>/dev/null
  (cd tools/ab_r1 && timeout 900 python bench.py --no-cpu-baseline --config C5 --gib 16 --page-size 4096 --steps 3 > ../../gpurun_out/r2zp_r1_c5p4k_$k.json 2>/dev/null)
  timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C5 --gib 16 --page-size 4096 --steps 3 --compress 0 > gpurun_out/r2zp_now_c5p4k_$k.json 2>/dev/null
  (cd tools/ab_r1 && timeout 900 python bench.py --no-cpu-baseline --config C4 --mode incremental --dirty 0.01 --steps 5 > ../../gpurun_out/r2zp_r1_c4_$k.json 2>/dev/null)
  timeout 900 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > gpurun_out/r2zp_now_c4_$k.json 2>/dev/null
done
