#!/bin/bash
# bench.py over the five BASELINE configs (config 1 and config 4 at each delta
# of their sweep) -> gpurun_out/configs/<name>_<delta>.json; summarise with
#    python profiles/configs_table.py gpurun_out/configs
mkdir -p gpurun_out/configs
run() {  # name delta
  timeout 900 python bench.py --config $1 --delta $2 --steps 3 --warmup 3 \
    > gpurun_out/configs/$1_$2.json 2> gpurun_out/configs/$1_$2.err
  echo "$1 delta $2 rc=$?"
}
run uniform_10k_200k 1000
run powerlaw_1m_10m 600
run powerlaw_1m_10m 3600
run powerlaw_1m_10m 86400
run hubstress_100k_50m 3600
run triadic_25m_100m 3600
run triadic_25m_100m 86400
run powerlaw_50m_600m 600
run powerlaw_50m_600m 3600
run powerlaw_50m_600m 86400
