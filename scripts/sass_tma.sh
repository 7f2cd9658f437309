#!/bin/bash
# TMA / mbarrier evidence from the built library's SASS (runs here, no GPU):
#   scripts/sass_tma.sh > profiles/r02_sass_tma.txt
# Per kernel: how many UBLKCP (1-D bulk copy), UTMALDG (tensor copy),
# SYNCS.ARRIVE (mbarrier arrive / expect_tx) and SYNCS.PHASECHK (mbarrier
# wait) instructions it holds; then the issue + wait sequence of k_detect_p8.
SO=${1:-paper_2412_15122_b200/libapsp_warm.so}
echo "# cuobjdump -sass $SO  ($(date -u +%F), $(/usr/local/cuda/bin/cuobjdump --version | tail -1))"
echo "# count  instruction  kernel"
/usr/local/cuda/bin/cuobjdump -sass "$SO" | awk '/Function :/{fn=$3} /UBLKCP|UTMALDG|SYNCS\.PHASECHK|SYNCS\.ARRIVE/{split($0,a,/ +/); for(i=1;i<=NF;i++) if ($i ~ /^(UBLKCP|UTMALDG|SYNCS)/) {c[fn"\t"$i]++; break}} END{for(k in c) print c[k]"\t"k}' \
  | sort -t$'\t' -k2,2 -k3,3 | while IFS=$'\t' read n fn ins; do printf "%3d  %-32s %s\n" "$n" "$ins" "$(echo "$fn" | c++filt | cut -c1-110)"; done
echo
echo "# k_detect_p8<int, false, 1>: the ring refill and wait (excerpt)"
/usr/local/cuda/bin/cuobjdump -sass -fun '_ZN4apsp11k_detect_p8IiLb0ELi1EEEvNS_4RowsElllNS_6TilingEPKT_S5_S5_S5_NS_9DetectOutIS3_EE14CUtensorMap_st' "$SO" 2>/dev/null \
  | grep -B2 "UTMALDG\|SYNCS.PHASECHK" | grep -v "^\s*/\* 0x" | sed 's/^\s*//; s/ *\/\* 0x[0-9a-f]* \*\/$//' | head -30
