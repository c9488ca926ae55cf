# round-2 GPU job 21: full GPU suite, bench lines (default, cfg1, reference arms), launch list of the default bench
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r02u_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/r02u_pytest_gpu.log; tail -5 $O/r02u_pytest_gpu.log
python bench.py > $O/r02u_bench_default.json 2> $O/r02u_bench_default.err; tail -c 600 $O/r02u_bench_default.json
python bench.py --impl reference > $O/r02u_bench_reference_arm.json 2> $O/r02u_bench_reference_arm.err; tail -c 600 $O/r02u_bench_reference_arm.json
python bench.py --workload cfg1 > $O/r02u_bench_cfg1.json 2> $O/r02u_bench_cfg1.err
python bench.py --workload cfg1 --impl reference > $O/r02u_bench_cfg1_reference_arm.json 2> $O/r02u_bench_cfg1_ref.err
python bench.py --steps 2 --warmup 1 --no-aesc --no-cpu-baseline > $O/r02u_plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02u_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-aesc --no-cpu-baseline > $O/r02u_ncu_launch.log 2>&1
python tools/launch_summary.py $O/r02u_launches_cfg2.csv > $O/r02u_launches_cfg2_summary.txt; cat $O/r02u_launches_cfg2_summary.txt
