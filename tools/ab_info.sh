#!/bin/bash
# Interleaved A/B of the config-2 GP-70 info build: in-tree library vs tuning variants
# (tools/build_variant.py), two rounds:  bash tools/ab_info.sh tune/a.so [tune/b.so ...]
for i in 1 2; do
  for v in base "$@"; do
    if [ $v = base ]; then unset FIF_LIB; else export FIF_LIB=$PWD/$v; fi
    echo "$v $(python tools/prof_build.py --kind ${KIND:-info} --reps 4 2>&1 | tail -1)"
  done
done
