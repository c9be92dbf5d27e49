nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 50 > /tmp/smi_d8.csv &
SMI=$!
GPB_OZAKI=8 N=32768 T=64 D=${D:-8} EXPORT=0 REPS=12 python tools/oz_chol_check.py 2>&1 | grep planes
kill $SMI
awk -F, '$2+0 > 350 {print $1, $3}' /tmp/smi_d8.csv | sort | uniq -c | sort -rn | head -5
awk -F, '$2+0 > 350 {s+=$2; n++} END {print "mean power under load", s/n, "W over", n, "samples"}' /tmp/smi_d8.csv
