# round-2 GPU job 6: suite, default bench (AESC roofline run), cfg1 line, cfg4/cfg5 AESC lines
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider -W "always::UserWarning" > $O/r02f_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02f_pytest.log
tail -4 $O/r02f_pytest.log
python bench.py > $O/r02f_bench.json 2> $O/r02f_bench.err; echo bench rc=$?
python bench.py --workload cfg1 > $O/r02f_bench_cfg1.json 2> $O/r02f_bench_cfg1.err; echo cfg1 rc=$?
python bench.py --impl reference --workload cfg1 > $O/r02f_bench_cfg1_ref.json 2> $O/r02f_bench_cfg1_ref.err; echo cfg1ref rc=$?
python bench.py --workload cfg5 > $O/r02f_bench_cfg5.json 2> $O/r02f_bench_cfg5.err; echo cfg5 rc=$?
python bench.py --workload cfg4 > $O/r02f_bench_cfg4.json 2> $O/r02f_bench_cfg4.err; echo cfg4 rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02f_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-aesc --no-cpu-baseline > $O/r02f_ncu_launch.log 2>&1
python tools/launch_summary.py $O/r02f_launches_cfg2.csv > $O/r02f_launches_cfg2_summary.txt; head -8 $O/r02f_launches_cfg2_summary.txt
