#!/bin/bash
# GPU check used between changes: the GPU test suite, then one bench line.
#   profiles/gpu_check.sh <tag>   (results in gpurun_out/<tag>/)
tag=${1:-check}
out=gpurun_out/$tag
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest=$?"
tail -2 $out/pytest.log
timeout 300 python bench.py > $out/bench.json 2> $out/bench.err; echo "bench=$?"
python - "$out/bench.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
r = d["roofline"]
print(f"value {d['value']/1e9:.3f} G edges/s  ms/step {d['ms_per_step']:.4f}  e2e {d['e2e']['value']/1e9:.3f}  "
      f"{r['kernel']} frac {r['frac']:.3f}  clocks {d['clocks']}")
PY
