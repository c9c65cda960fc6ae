#!/bin/bash
# Interleaved step times of several library builds on one box:
#   profiles/abn.sh ROUNDS "bench args" lib1.so lib2.so ...   ("" = the in-tree build)
N=$1; ARGS=$2; shift 2
for i in $(seq "$N"); do
  for lib in "$@"; do
    TM_LIB=$lib python bench.py --no-cpu-baseline --no-reader --steps 20 $ARGS 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-tree}', round(d['ms_per_step'],4))"
  done
done
