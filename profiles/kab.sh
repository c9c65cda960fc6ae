#!/bin/bash
# Interleaved per-kernel times (CUDA events, serialised) of several library
# builds on one box:  profiles/kab.sh ROUNDS CONFIG DELTA lib1.so lib2.so ...
#   ("" = the in-tree build); one JSON line per (round, lib)
N=$1; CFG=$2; D=$3; shift 3
for i in $(seq "$N"); do
  for lib in "$@"; do
    TM_LIB=$lib KTIMES=1 timeout 900 python profiles/census_once.py $CFG $D 2 2>/dev/null |
      python -c "
import json,sys
L=[json.loads(x) for x in sys.stdin if x.strip()]
k=[x for x in L if 'kernel_ms' in x]
r=[x for x in L if 'rep' in x]
print(json.dumps({'lib':'${lib:-tree}','round':$i,'s':[x['s'] for x in r],'total':r[-1]['census_total'] if r else None,'kernel_ms':k[0]['kernel_ms'] if k else None}))"
  done
done
