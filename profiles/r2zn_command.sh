#!/bin/bash
# chunk size for incremental checkpoints: 256 / 512 / 1024 MiB on C4 1 % at 8 and 40 GiB, and C2 f4 (full)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2zn_build.log 2>&1
for k in 1 2; do for C in 1024 512 256; do
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --gib 8 --mode incremental --dirty 0.01 --steps 10 --compress 0 --chunk-mb $C > gpurun_out/r2zn_c4g8_c${C}_$k.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 5 --compress 0 --chunk-mb $C > gpurun_out/r2zn_c4_c${C}_$k.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --steps 5 --chunk-mb $C > gpurun_out/r2zn_c2_c${C}_$k.json 2>/dev/null
done; done
