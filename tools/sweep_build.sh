#!/bin/bash
# Config-2 GP build timings of the in-tree library and tuning variants (tools/build_variant.py):
#   bash tools/sweep_build.sh tune/a.so tune/b.so ...
for v in base "$@"; do
  if [ $v = base ]; then unset FIF_LIB; else export FIF_LIB=$PWD/$v; fi
  echo "== $v"
  python tools/prof_build.py --kind trace --reps 3 2>&1 | tail -1
  python tools/prof_build.py --kind info --reps 3 2>&1 | tail -1
done
