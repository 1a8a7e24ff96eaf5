#!/bin/bash
# HEAD confirmation after the container re-creation: smoke, every GPU test, the
# default bench line; plus a GCR_TRACE timeline of the C4 1 % incremental step
# and of the 8 GiB sub-record shape (pipeline study)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2t_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
GCR_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --gib 8 --mode incremental --dirty 0.01 --steps 3 --compress 0 > gpurun_out/r2t_c4g8.json 2> gpurun_out/r2t_c4g8_trace.err
GCR_TRACE=1 timeout 600 python bench.py --no-cpu-baseline --sub-c4-gib 0 --config C4 --mode incremental --dirty 0.01 --steps 3 --compress 0 > gpurun_out/r2t_c4.json 2> gpurun_out/r2t_c4_trace.err
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/r2t_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2t_gputests.log
