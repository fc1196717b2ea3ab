#!/bin/bash
# SASS instruction census of the library (tensor-core / async-copy evidence per kernel family)
LIB=${1:-paper_2109_05451_b200/libh2b200.so}
cuobjdump -sass "$LIB" > /tmp/h2_sass.txt
echo "# SASS census of $(basename $LIB) ($(date -u +%F))"
for op in DMMA.8x8x4 HMMA.1688.F32.TF32 UTCHMMA UTMALDG UBLKCP LDTM UTCBAR DFMA FFMA LDGSTS SYNCS.ARRIVE SYNCS.PHASECHK LDS STS SHFL RED.E.ADD ATOMG; do
  printf "%-16s %8d\n" "$op" "$(grep -c "$op" /tmp/h2_sass.txt)"
done
echo "# per kernel (DMMA / HMMA-TF32 / UTCHMMA / UTMALDG / LDGSTS / UBLKCP / FFMA / DFMA)"
awk '/Function :/{f=$3} /DMMA/{d[f]++} /HMMA.*TF32/{h[f]++} /UTCHMMA/{t[f]++} /UTMALDG/{m[f]++} /LDGSTS/{g[f]++} /UBLKCP/{u[f]++} /FFMA/{s[f]++} /DFMA/{df[f]++} END{for (k in d) seen[k]=1; for (k in h) seen[k]=1; for (k in t) seen[k]=1; for (k in g) seen[k]=1; for (k in s) seen[k]=1; for (k in df) seen[k]=1; for (k in seen) printf "%6d %6d %6d %6d %6d %6d %6d %6d %s\n", d[k], h[k], t[k], m[k], g[k], u[k], s[k], df[k], k}' /tmp/h2_sass.txt | sort -k9 | c++filt | cut -c1-200
