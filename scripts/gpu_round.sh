#!/bin/bash
# Round evidence on one B200 (outputs under gpurun_out/): smoke, the full GPU suite, the bench line,
# the serialised launch list of a c3 solve.  SKIP_TESTS / SKIP_BENCH / SKIP_LAUNCHES skip parts.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
if [ -z "$SKIP_TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
  tail -3 gpurun_out/pytest_gpu.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
  head -c 400 gpurun_out/bench.json; echo
fi
if [ -z "$SKIP_LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 1500 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --cpu-baseline-iters 0 --no-e2e --no-p3 \
    --kernel-reps 2 --host-loop > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
fi
