#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v17_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v17_gputests.log 2>&1; echo rc=$? >> gpurun_out/v17_gputests.log
timeout 400 python bench.py > gpurun_out/v17_bench.json 2> gpurun_out/v17_bench.err
timeout 300 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 5 --no-cpu-baseline > gpurun_out/v17_c4.json 2> gpurun_out/v17_c4.err
