#!/bin/bash
# GEMM configuration sweep (standalone kernel timings + bitwise fingerprints)
for c in 4 5 8 9; do
  echo "== cfg $c"; GPB_GEMM_CFG=$c timeout 120 ./tools/gemm_bench
done
