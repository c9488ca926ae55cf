# round-2 GPU job 5: full GPU suite (compiled-reference full-size parity), bench, AESC timings, launch list
set -x
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider -W "always::UserWarning" --durations=15 > $O/r02e_pytest.log 2>&1; echo "pytest rc=$?" >> $O/r02e_pytest.log
tail -40 $O/r02e_pytest.log
python bench.py > $O/r02e_bench.json 2> $O/r02e_bench.err; echo bench rc=$?
for c in cfg3; do python tools/aesc_run.py --workload $c --reps 2 > $O/r02e_aesc_$c.log 2>&1; grep "^aesc:" $O/r02e_aesc_$c.log; done
python tools/aesc_run.py --workload cfg4 --sources 64 --reps 2 > $O/r02e_aesc_cfg4.log 2>&1; grep "^aesc:" $O/r02e_aesc_cfg4.log
python tools/aesc_run.py --workload cfg5 --sources 512 --reps 2 > $O/r02e_aesc_cfg5.log 2>&1; grep "^aesc:" $O/r02e_aesc_cfg5.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02e_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-aesc --no-cpu-baseline > $O/r02e_ncu_launch.log 2>&1
python tools/launch_summary.py $O/r02e_launches_cfg2.csv | head -12
