#!/bin/bash
# sweep GEMM kernel configurations on the config-2 bench
for c in 0 1 2 3; do
  GPB_GEMM_CFG=$c timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/sweep_$c.json 2>gpurun_out/sweep_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/sweep_$c.json'))
print('cfg $c', round(d['value'],2), 'TF chol |', round(d['predict_variance']['value']), 'pts/s |', {k: round(v,1) for k,v in d['phases_ms_per_step'].items()}, '| gemm', round(d['roofline']['achieved'],2))"
done
