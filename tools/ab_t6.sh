#!/bin/bash
# Interleaved A/B of the config-2 GP-70 info build (k_gp_info_t6 variants), with a precision
# check of every variant first:  bash tools/ab_t6.sh tune/a.so [tune/b.so ...]
for v in base "$@"; do
  if [ $v = base ]; then unset FIF_LIB; else export FIF_LIB=$PWD/$v; fi
  echo "== $v"; KERNELS=t6,h16 timeout 300 python tools/t5_probe.py 2>&1 | grep -E "^t6"
done
for i in 1 2; do
  for v in base "$@"; do
    if [ $v = base ]; then unset FIF_LIB; else export FIF_LIB=$PWD/$v; fi
    echo "$v $(python tools/prof_build.py --kind info --reps 4 2>&1 | tail -1)"
  done
done
