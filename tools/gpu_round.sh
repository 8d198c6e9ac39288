# Round measurement (run under gpurun from the repo root): GPU tests, smoke, both bench arms,
# the ncu launch list of the bench command and one --set full capture of the headline kernel
# (each ncu pass only after the same command exited 0 without ncu).
set -x
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gputest.log 2>&1; echo GPUTEST_RC=$? >> $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo SMOKE_RC=$? >> $O/smoke.log
python bench.py > $O/bench.json 2> $O/bench.err; echo BENCH_RC=$?
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo REF_RC=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_small.json 2> $O/bench_small.err && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo NCU1=$?
python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > $O/bench_tiny.json 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_gp_info_t5 -s 2 -c 1 -f -o $O/t5_bench_full python bench.py --steps 1 --warmup 3 --no-extras --no-cpu-baseline > $O/ncu_full.log 2>&1; echo NCU2=$?
tail -2 $O/gputest.log; tail -1 $O/smoke.log
