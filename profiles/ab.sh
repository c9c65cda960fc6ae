#!/bin/bash
# A/B step time of two library builds on the same box, interleaved:
#   profiles/ab.sh ab/lib_prev.so [rounds] [bench args...]
A=${1:?lib}; N=${2:-3}; shift 2
for i in $(seq "$N"); do
  for lib in "$A" ""; do
    TM_LIB=$lib python bench.py --no-cpu-baseline --steps 20 "$@" 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-new}', round(d['ms_per_step'],4))"
  done
done
