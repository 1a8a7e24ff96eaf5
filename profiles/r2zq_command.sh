#!/bin/bash
# does the f1 (in-scan pack) code in K1 cost the default path?  K1 built with
# the f1 hooks compiled out (tools/ab_noisp) vs the current code, alternating:
# C4 1 % (incremental K1) and C2 (full K1, K8)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2zq_build.log 2>&1
(cd tools/ab_noisp && python -c "import __graft_entry__ as g; g.build()") >> gpurun_out/r2zq_build.log 2>&1
for k in 1 2; do
  (cd tools/ab_noisp && timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > ../../gpurun_out/r2zq_noisp_c4_$k.json 2>/dev/null)
  timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 > gpurun_out/r2zq_now_c4_$k.json 2>/dev/null
  (cd tools/ab_noisp && timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --steps 10 --compress 0 > ../../gpurun_out/r2zq_noisp_c2_$k.json 2>/dev/null)
  timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --steps 10 --compress 0 > gpurun_out/r2zq_now_c2_$k.json 2>/dev/null
done
