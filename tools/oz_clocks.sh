#!/bin/bash
# SM clock, throttle reason and power while the digit-plane product runs alone, back to
# back for a few seconds (long-k shape, 8 planes): is it power-capped when sustained?
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Iinclude -Ipaper_2505_00136_b200/csrc \
  -o /tmp/ozaki_probe tools/ozaki_probe.cu paper_2505_00136_b200/csrc/ozaki.cu -lcuda
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 50 > /tmp/smi_probe.csv &
SMI=$!
/tmp/ozaki_probe time ${REPS:-400} | tail -2
kill $SMI
awk -F, '$2+0 > 400 {print $1, $3}' /tmp/smi_probe.csv | sort | uniq -c | sort -rn | head -6
awk -F, '$2+0 > 400 {s+=$2; n++} END {print "mean power under load", s/n, "W over", n, "samples"}' /tmp/smi_probe.csv
