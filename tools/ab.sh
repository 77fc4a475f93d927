#!/bin/bash
# A/B timing of variant libraries, interleaved over rounds; prints the median GB/s per
# (library, m).   tools/ab.sh "lib variants/x.so" "4,8,16" 5 [extra scan_one args]
LIBS=$1; MS=$2; ROUNDS=${3:-5}; shift 3
for r in $(seq $ROUNDS); do
  for v in $LIBS; do
    if [ "$v" = lib ]; then L=""; else L="--lib $v"; fi
    python tools/scan_one.py $L --m $MS --reps 7 "$@"
  done
done | python3 -c '
import sys, re, statistics, collections
d = collections.defaultdict(list)
for line in sys.stdin:
    m = re.match(r"(\S+) m=(\d+) ms=\S+ GB/s=(\S+)", line)
    if m:
        d[(m.group(1), int(m.group(2)))].append(float(m.group(3)))
libs = sorted({k[0] for k in d}); ms = sorted({k[1] for k in d})
print("m      " + "  ".join(f"{l[-14:]:>14s}" for l in libs))
for mm in ms:
    print(f"{mm:<6d} " + "  ".join(f"{statistics.median(d[(l, mm)]):14.0f}" for l in libs))
'
