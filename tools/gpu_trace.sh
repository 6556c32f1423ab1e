# needs a library built with the timeline compiled in: bash tools/ab_defines.sh T "-DBNFF_WC_TRACE=1"
for c in 29 27 28 26 33; do echo "=== case $c"; BNFF_LIB=$PWD/paper_1807_01702_b200/libbnff_T.so timeout 120 python tools/trace_conv.py --only $c 2>&1 | grep -v "RuntimeWarning\|nanmean\|print(" | tail -22 | head -12; done
