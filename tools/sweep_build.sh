#!/bin/bash
O=gpurun_out; mkdir -p $O
for v in base tune/v_t0.so tune/v_t1.so tune/v_m2.so tune/v_m4.so; do
  if [ $v = base ]; then unset FIF_LIB; else export FIF_LIB=$PWD/$v; fi
  echo "== $v"
  python tools/prof_build.py --kind trace --reps 3 2>&1 | tail -1
  python tools/prof_build.py --kind info --reps 3 2>&1 | tail -1
done
unset FIF_LIB
python tools/perf_probe.py 2>&1 | head -8
