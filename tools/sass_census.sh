#!/bin/bash
# SASS instruction census of the executor library (proof of the tcgen05 /
# TMA / TMEM paths): per kernel family, counts of the mnemonics
# B200_PROFILING.md names. Usage: tools/sass_census.sh > profiles/rNN/sass_census.txt
so=${1:-paper_2301_08984_b200/_lib/libplanc_b200.so}
tmp=$(mktemp)
cuobjdump -sass "$so" > "$tmp"
echo "# cuobjdump -sass $so ($(date -u +%F))"
echo "# whole library"
for m in UTCHMMA UTCQMMA UTCMMA UTMALDG UTMASTG UTMAPF UBLKCP LDTM STTM UTCBAR HMMA FFMA STL LDL; do
  printf "%-10s %8d\n" $m "$(grep -cE "\b$m(\.|\b)" "$tmp")"
done
echo "# 2-SM (cta_group::2) MMAs"
printf "%-10s %8d\n" UTCHMMA.2CTA "$(grep -cE 'UTCHMMA\.2CTA' "$tmp")"
echo "# per kernel (functions with any tcgen05 / TMA instruction)"
awk '/Function :/{f=$3} /UTCHMMA|UTMALDG|UTMASTG|LDTM/{c[f]++} END{for(k in c) printf "%8d  %s\n", c[k], k}' "$tmp" | sort -rn | head -40
rm -f "$tmp"
