#!/bin/bash
# K1 L2-prefetch distance sweep (scratch experiment)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pf_parity.log 2>&1; echo rc=$? >> gpurun_out/pf_parity.log
: > gpurun_out/pf_sweep.jsonl
for pf in 0 4096 8192 16384 32768; do
  for cfg in "--config C2 --steps 5" "--config C4 --mode incremental --dirty 0.01 --steps 4 --chunk-mb 1024"; do
    line=$(GCR_SCAN_PREFETCH=$pf timeout 300 python bench.py --no-cpu-baseline $cfg 2>>gpurun_out/pf_sweep.err | tail -1)
    python -c "import json,sys; d=json.loads(sys.argv[1]); print(json.dumps({'pf':int(sys.argv[2]),'cfg':sys.argv[3],'value':d['value'],'ms':d['ms_per_step'],'k1':d['kernels']['K1_scan'],'k8':d['kernels']['K8_verify'],'roof':d['roofline']['frac']}))" "$line" $pf "$cfg" >> gpurun_out/pf_sweep.jsonl
  done
done
