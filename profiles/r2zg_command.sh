#!/bin/bash
# why K1 trails K8 on C2 at 2 MiB pages: chunk size (1 vs 2 chunks) and page size A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2zg_build.log 2>&1
for P in 2097152 65536; do for C in 2048 1024 512; do
timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --compress 0 --page-size $P --chunk-mb $C --steps 5 > gpurun_out/r2zg_p${P}_c${C}.json 2>/dev/null
done; done
