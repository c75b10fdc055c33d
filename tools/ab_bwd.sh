#!/bin/bash
# A/B the backward kernel variants in build/variants: ROUNDS alternating passes of
# tools/probe_bwd_perf.py per variant, then the median TFLOP/s per (variant, case).
# usage: tools/ab_bwd.sh v1 v2 ...   (ROUNDS=3 by default)
R=${ROUNDS:-3}
out=$(mktemp)
for r in $(seq $R); do
  for v in "$@"; do
    ZP_LIB_PATH=$PWD/build/variants/$v.so timeout 120 python tools/probe_bwd_perf.py 2>&1 | \
      sed -n "s/^bwd seqlens=\(\[[^]]*\]\).*TFLOP\/s=\([0-9.]*\).*/$v \1 \2/p" >> $out
  done
done
python - "$out" <<'PY'
import sys, collections, statistics
d = collections.defaultdict(list)
for line in open(sys.argv[1]):
    v, rest = line.split(' ', 1)
    case, val = rest.rsplit(' ', 1)
    d[(case, v)].append(float(val))
for (case, v), xs in sorted(d.items()):
    print(f"{case:32s} {v:14s} median {statistics.median(xs):7.1f}  all {xs}")
PY
