#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/v20.jsonl
for v in t640_u5 t512_u8 t512_u6 t640_u6 t768_u4; do
  GCR_LIBRARY=$PWD/scratch/libgcr_$v.so timeout 300 python scratch/scan_size.py 2>/dev/null | sed "s/^{/{\"var\": \"$v\", /" >> gpurun_out/v20_scan.jsonl
  line=$(GCR_LIBRARY=$PWD/scratch/libgcr_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); k=d['kernels']; print(json.dumps({'var':sys.argv[2],'run':'c2','K1':k['K1_scan']['GBps'],'K8':k['K8_verify']['GBps'],'roof':d['roofline']['frac']}))" "$line" $v >> gpurun_out/v20.jsonl
  line=$(GCR_LIBRARY=$PWD/scratch/libgcr_$v.so timeout 300 python bench.py --config C4 --mode incremental --dirty 0.01 --steps 4 --no-cpu-baseline 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); k=d['kernels']; print(json.dumps({'var':sys.argv[2],'run':'c4','K1':k['K1_scan']['GBps'],'ms':d['ms_per_step']}))" "$line" $v >> gpurun_out/v20.jsonl
done
