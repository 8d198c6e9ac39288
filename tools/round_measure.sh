#!/bin/bash
# Round-end measurement recipe (run under gpurun from the repo root).
# Each ncu pass runs only after the same command exited 0 without ncu.  The --set full
# reports are summarised on the box (text + ncu_summary.json) and only the headline
# kernel's report is kept, so gpurun_out/ stays under the 64 MiB copy-back limit.
set -u
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
python bench.py > $O/bench.json 2> $O/bench.err || exit 1
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_short.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/prof_build.py --kind trace > $O/trace_build.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_gp_trace -c 1 -o $O/full_k_gp_trace -f \
      python tools/prof_build.py --kind trace --reps 1 > $O/ncu_full_k_gp_trace.log 2>&1
for k in k_gp_info_h16 k_query_info k_pc_fim k_query_prep_gp; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o $O/full_$k -f \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_full_$k.log 2>&1
done
python tools/ncu_json.py $O $O/ncu_summary.json > $O/ncu_json.log 2>&1
for k in k_gp_info_h16 k_gp_trace k_query_info k_query_prep_gp k_pc_fim; do
  echo "== $k"; python tools/ncu_summary.py $O/full_$k.ncu-rep $k
done > $O/ncu_full_summary.txt 2>&1
for k in k_gp_trace k_query_info k_query_prep_gp k_pc_fim; do rm -f $O/full_$k.ncu-rep; done
