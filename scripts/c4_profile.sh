#!/bin/bash
# c4 (Oseen n = 512, two-stage PCD) timing and serialised launch list (outputs under gpurun_out/)
timeout 600 python scripts/run_configs.py --only c4,c4s > gpurun_out/c4_configs.json 2> gpurun_out/c4_configs.err; echo c4=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
  --log-file gpurun_out/c4_launches.csv python scripts/run_configs.py --only c4 > gpurun_out/c4_ncu.log 2>&1; echo c4_launches=$?
