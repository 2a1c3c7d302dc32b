#!/bin/bash
# Round evidence on one B200: bench line, serialised launch list of a c3 solve, full ncu captures
# of the dominant kernels.  Outputs under gpurun_out/ (copy what is judged into profiles/).
set -x
[ -n "$SKIP_BENCH" ] || timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 1500 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --cpu-baseline-iters 0 --no-e2e --no-p3 \
  --kernel-reps 2 --host-loop > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
[ -n "$SKIP_NCU" ] || for k in "k_sgs_tile:10" "k_cheb_tile:11" "k_saddle_tile:0"; do
  name=${k%%:*}; which=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name -s 2 -c 1 \
    -o gpurun_out/$name python scripts/profile_kernel.py --n 1024 --which $which --reps 2 > gpurun_out/ncu_$name.log 2>&1
  echo ncu_$name=$?
done
