#!/bin/bash
# c4 (Oseen n = 512, two-stage PCD) timing and serialised launch list of the solve (setup launches
# skipped; outputs under gpurun_out/)
timeout 600 python scripts/run_configs.py --only c4,c4s > gpurun_out/c4_configs.json 2> gpurun_out/c4_configs.err; echo c4=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip ${C4_SKIP:-13500} -c ${C4_COUNT:-30000} --csv \
  --log-file gpurun_out/c4_launches.csv python scripts/c4_ab.py > gpurun_out/c4_ncu.log 2>&1; echo c4_launches=$?
