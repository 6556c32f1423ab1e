for c in 29 27 28 26 33; do echo "=== case $c"; timeout 120 python tools/trace_conv.py --only $c 2>&1 | grep -v "RuntimeWarning\|nanmean\|print(" | tail -22 | head -12; done
