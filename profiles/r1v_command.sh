#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v19_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/v19_gputests.log 2>&1; echo rc=$? >> gpurun_out/v19_gputests.log
timeout 400 python bench.py > gpurun_out/v19_bench.json 2> gpurun_out/v19_bench.err
