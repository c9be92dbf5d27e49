#!/bin/bash
# TMA-fed GEMM vs the cp.async kernel (standalone timings + fingerprints)
for m in 0 1 2 3; do
  echo "== GPB_GEMM_TMA=$m"; GPB_GEMM_TMA=$m timeout 120 ./tools/gemm_bench
done
