for c in 25 23; do echo "=== case $c"; timeout 120 python tools/trace_conv.py --only $c 2>&1 | tail -24 | head -12; done
