set -x
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo GPUTEST_RC=$? >> gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_RC=$? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH_RC=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo NCU1=$?
python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_tiny.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gp_info_t5 -s 2 -c 1 -o gpurun_out/t5_bench_full python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo NCU2=$?
tail -2 gpurun_out/gputest.log; tail -1 gpurun_out/smoke.log
