# Round measurement: bench line (ours + reference arm), launch list, ncu --set full of the
# headline kernel, the PC kernel and the query contraction (each after a clean plain run)
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH_RC=$?
python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo REF_RC=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo NCU1=$?
python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_tiny.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gp_info_t5 -s 2 -c 1 -o gpurun_out/r02_t5_full python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo NCU2=$?
python tools/prof_pc.py --poses 1000000 --reps 2 > gpurun_out/pc_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pc_fim -s 1 -c 1 -o gpurun_out/r02_pc_full python tools/prof_pc.py --poses 1000000 --reps 2 > gpurun_out/ncu_pc.log 2>&1; echo NCU3=$?
python tools/prof_query.py --reps 3 > gpurun_out/q_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_query_info|k_query_prep_gp" -s 2 -c 2 -o gpurun_out/r02_query_full python tools/prof_query.py --reps 3 > gpurun_out/ncu_q.log 2>&1; echo NCU4=$?
